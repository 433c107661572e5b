#!/bin/bash
# Fig. 5 reproduction: timing run + per-method ncu DRAM-traffic pass (one call each).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wl in ${WLS:-vlm64k dit64k}; do
  timeout -s KILL 600 python scripts/fig5.py --workload $wl > gpurun_out/fig5_$wl.log 2>&1; tail -1 gpurun_out/fig5_$wl.log
  for m in fused_alg1 fused_exact naive_mins naive_topp; do
    timeout -s KILL 600 /usr/local/cuda/bin/ncu --profile-from-start off --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      --log-file gpurun_out/fig5_${wl}_$m.csv python scripts/fig5.py --workload $wl --method $m --once \
      > gpurun_out/fig5_${wl}_$m.log 2>&1
  done
done
