#!/bin/bash
# P_q / B_K / G_K latency ablation at matched sparsity (alpha calibrated
# per point), dit128k (non-causal) and vlm64k (causal).  Kernel-only bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-abl_r01}
OUT=gpurun_out/sweep_$TAG.jsonl
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {
  timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --no-context --no-causal-extra --steps 3 --warmup 3 --dense-reps 0 "$@" 2>>gpurun_out/sweep_$TAG.err | tail -1 >> $OUT
}
for wl in dit128k vlm64k; do
  for pq in 64 128; do run --workload $wl --pq $pq; done
  for bk in 32 64; do run --workload $wl --bk $bk; done
  for gk in 1 16 256 8192; do run --workload $wl --gk $gk; done
done
wc -l $OUT
