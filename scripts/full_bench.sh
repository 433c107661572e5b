#!/bin/bash
# Full bench (ours + reference arm), the ncu launch list of the same command, and one
# full-size `ncu --set full` capture of the sparse attention kernel (-> traffic).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NO_NCU" ]; then
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --alpha 1.0039 --dense-reps 1 --no-context --no-causal-extra \
  > gpurun_out/launches_$TAG.log 2>&1
# full-size sparse kernel (fused forward, 24 heads): 1 select pass then the attention launch
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_db_kernel -s 0 -c 1 \
  -o gpurun_out/prof_$TAG -f python scripts/prof_run.py --reps 1 --no-dense --fused > gpurun_out/prof_$TAG.log 2>&1
python scripts/summarize_ncu.py $TAG > /dev/null 2>&1
# selection kernel and dense kernel (--set full, one launch each)
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"select_kernel|attn_kernel" -s 0 -c 2 \
  -o gpurun_out/prof_${TAG}_extra -f python scripts/prof_run.py --reps 1 > gpurun_out/prof_${TAG}_extra.log 2>&1
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -1 gpurun_out/bench_ref_$TAG.json
