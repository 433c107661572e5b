#!/bin/bash
# Full bench (ours + reference arm) and the ncu launch list of the same command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -1 gpurun_out/bench_ref_$TAG.json
if [ -z "$NO_NCU" ]; then
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --alpha 1.0039 --dense-reps 1 \
  > gpurun_out/launches_$TAG.log 2>&1
TAG=$TAG KREGEX=attn_kernel SKIP=2 COUNT=2 ARGS="--heads 4 --reps 2" bash scripts/profile_one.sh
fi
