#!/bin/bash
# A/B of two versions of one kernel source on the same box, runs interleaved A B A B ...
# usage: scripts/ab.sh <csrc file name> <dir with A_<name>, B_<name>> [rounds]
cd "$(dirname "$0")/.."
f=$1; d=$2; n=${3:-2}
mkdir -p gpurun_out/ab
for v in A B; do
  cp "$d/${v}_$f" paper_2603_29494_b200/csrc/$f
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build_$v.log 2>&1 || { tail -5 gpurun_out/ab/build_$v.log; exit 1; }
  cp paper_2603_29494_b200/libvecattn.so gpurun_out/ab/lib_$v.so
done
for i in $(seq $n); do for v in A B; do
  cp gpurun_out/ab/lib_$v.so paper_2603_29494_b200/libvecattn.so
  timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline ${ALPHA_ARGS:---alpha 1.0039} --dense-reps 0 ${BENCH_ARGS} > gpurun_out/ab/b.json 2>gpurun_out/ab/b_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab/b.json').read().strip().splitlines()[-1]); print('$v', d['stage_ms'].get('attention'), d['forward_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab/b_$v.err
done; done
