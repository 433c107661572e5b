#!/bin/bash
# SURVEY.md 8(d) sweep on one GPU: named configs, rho grid and N sweep (kernel-only bench lines).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
OUT=gpurun_out/sweep_$TAG.jsonl
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {
  timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --no-context --no-causal-extra --steps 3 --warmup 3 --dense-reps 1 "$@" 2>>gpurun_out/sweep_$TAG.err | tail -1 >> $OUT
}
run --workload dit128k --rho 0.785
run --workload vlm128k --rho 0.785
run --workload vlm64k --rho 0.785
run --workload hy --rho 0.621
run --workload hy --rho 0.785
run --workload wan --rho 0.523
run --workload dit128k --rho 0.785 --kind gauss
run --workload dit128k --rho 0.785 --mode exact
run --workload dit128k --rho 0.785 --mode topk
for r in 0.5 0.75 0.9 0.93 0.95; do run --workload dit128k --rho $r; done
for n in 16 32 64 256; do run --workload dit${n}k --rho 0.785; done
for n in 16 32 64; do run --workload vlm${n}k --rho 0.785; done
wc -l $OUT
