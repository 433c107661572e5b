#!/bin/bash
# A/B of attn.cu variants on the dense denominator and the causal sparse path:
#   abdense.sh <rounds> tag ...   (prebuilt by scripts/build_variant.py; "main" = in-tree)
cd "$(dirname "$0")/.."
n=$1; shift
mkdir -p gpurun_out/ab
cp paper_2603_29494_b200/libvecattn.so gpurun_out/ab/lib_main.so
for i in $(seq $n); do for v in "$@"; do
  if [ "$v" = main ]; then cp gpurun_out/ab/lib_main.so paper_2603_29494_b200/libvecattn.so; else cp paper_2603_29494_b200/build/ab/lib_$v.so paper_2603_29494_b200/libvecattn.so; fi
  timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --alpha 1.0039 --dense-reps 2 --no-context --no-causal-extra --steps 2 > gpurun_out/ab/d.json 2>gpurun_out/ab/d_$v.err
  timeout -s KILL 300 python bench.py --workload vlm128k --no-e2e --no-cpu-baseline --alpha 0.39844 --dense-reps 2 --no-context --no-causal-extra --steps 3 > gpurun_out/ab/c.json 2>gpurun_out/ab/c_$v.err
  python -c "
import json
d=json.loads(open('gpurun_out/ab/d.json').read().strip().splitlines()[-1]); c=json.loads(open('gpurun_out/ab/c.json').read().strip().splitlines()[-1])
print('$v', 'dense128k', d['dense_ms'], 'sparse', d['forward_ms'], '| causal attn', c['stage_ms']['attention'], 'causal dense', c['dense_ms'], d['clocks']['sm_mhz'])" || { tail -3 gpurun_out/ab/d_$v.err; tail -3 gpurun_out/ab/c_$v.err; }
done; done
cp gpurun_out/ab/lib_main.so paper_2603_29494_b200/libvecattn.so
