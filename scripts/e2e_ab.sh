#!/bin/bash
# A/B of the e2e group ramp: e2e_ab.sh "1,2,4,7,7,2,1" "2,4,8,8,2" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
for i in 1 2; do for g in "$@"; do
  BENCH_E2E_GROUPS=$g timeout -s KILL 300 python bench.py --no-cpu-baseline --alpha 1.0039 --dense-reps 0 --no-context --no-causal-extra > gpurun_out/ab/e.json 2>gpurun_out/ab/e.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab/e.json').read().strip().splitlines()[-1]); print('$g', 'fwd', d['forward_ms'], 'e2e', round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab/e.err
done; done
