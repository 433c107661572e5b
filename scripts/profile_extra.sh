#!/bin/bash
# ncu --set full captures beyond the sparse attention: the selection GEMM/filter kernel and
# the dense kernel at dit128k, and the causal gather kernel at vlm128k (one launch each).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NCU="timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on"
$NCU -k regex:select_kernel -s 0 -c 1 -o gpurun_out/prof_${TAG}_select -f python scripts/prof_run.py --reps 1 --no-dense --fused > gpurun_out/prof_${TAG}_select.log 2>&1
$NCU -k regex:^attn_kernel -s 0 -c 1 -o gpurun_out/prof_${TAG}_dense -f python scripts/prof_run.py --reps 1 --heads 4 > gpurun_out/prof_${TAG}_dense.log 2>&1
$NCU -k regex:^attn_kernel -s 0 -c 1 -o gpurun_out/prof_${TAG}_causal -f python scripts/prof_run.py --reps 1 --no-dense --fused --workload vlm128k --alpha 0.39 > gpurun_out/prof_${TAG}_causal.log 2>&1
ls -la gpurun_out/prof_${TAG}_*
