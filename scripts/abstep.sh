#!/bin/bash
# Interleaved full-step A/B: abstep.sh <rounds> tag[:ENV=VAL] ...  (prebuilt build/ab/lib_<tag>.so; "main" = the tree's lib)
cd "$(dirname "$0")/.."
n=$1; shift
cp paper_2603_29494_b200/libvecattn.so /tmp/lib_main.so
for i in $(seq $n); do for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  if [ "$v" = main ]; then cp /tmp/lib_main.so paper_2603_29494_b200/libvecattn.so; else cp paper_2603_29494_b200/build/ab/lib_$v.so paper_2603_29494_b200/libvecattn.so; fi
  env $envs timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --no-context --no-causal-extra --alpha 1.0039 --dense-reps 0 > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$spec', 'step', d['ms_per_step'], 'stages', [round(d['stage_ms'][k],2) for k in ('select','emit_plan','attention')], d['clocks']['sm_mhz'])" || echo "$spec FAILED"
done; done
cp /tmp/lib_main.so paper_2603_29494_b200/libvecattn.so
