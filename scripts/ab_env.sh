#!/bin/bash
# A/B of runtime variants of the built library on one box, interleaved A B A B ...
# usage: scripts/ab_env.sh "<env A>" "<env B>" [rounds]   (e.g. "" "VECATTN_GATHER4=1")
cd "$(dirname "$0")/.."
A=$1; B=$2; n=${3:-2}
mkdir -p gpurun_out/ab
for i in $(seq $n); do for v in A B; do
  if [ $v = A ]; then E=$A; else E=$B; fi
  env $E timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline ${ALPHA_ARGS:---alpha 1.0039} --dense-reps 0 ${BENCH_ARGS} > gpurun_out/ab/b.json 2>gpurun_out/ab/b_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab/b.json').read().strip().splitlines()[-1]); print('$v [$E]', d['stage_ms'], d['forward_ms'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/ab/b_$v.err
done; done
