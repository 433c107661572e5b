#!/bin/bash
# Interleaved A/B of prebuilt library variants with per-variant env:
#   abvar.sh <rounds> tag[:ENV=VAL[,ENV2=VAL]] ...   (tag "main" = the in-tree build)
cd "$(dirname "$0")/.."
n=$1; shift
mkdir -p gpurun_out/ab
cp paper_2603_29494_b200/libvecattn.so gpurun_out/ab/lib_main.so
for i in $(seq $n); do for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
  if [ "$v" = main ]; then cp gpurun_out/ab/lib_main.so paper_2603_29494_b200/libvecattn.so; else cp paper_2603_29494_b200/build/ab/lib_$v.so paper_2603_29494_b200/libvecattn.so; fi
  env $envs timeout -s KILL 200 python bench.py --no-e2e --no-cpu-baseline ${ALPHA_ARGS:---alpha 1.0039} --dense-reps 0 ${BENCH_ARGS} > gpurun_out/ab/b.json 2>gpurun_out/ab/b_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab/b.json').read().strip().splitlines()[-1]); s=d['stage_ms']; print('$spec', 'attn', s.get('attention'), 'plan', s.get('emit_plan'), 'fwd', d['forward_ms'], d['clocks']['sm_mhz'])" || { echo "$spec FAILED"; tail -3 gpurun_out/ab/b_$v.err; }
done; done
cp gpurun_out/ab/lib_main.so paper_2603_29494_b200/libvecattn.so
