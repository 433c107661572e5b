#!/bin/bash
# Round-2 iteration: GPU tests (bounded), then bench A/B (pair kernel vs VECATTN_NO_PAIR).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-iter}
if [ "${TESTK:-all}" != none ]; then timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "${TESTK:-}" > gpurun_out/tests_$TAG.log 2>&1; tail -4 gpurun_out/tests_$TAG.log; fi
for v in ${VARIANTS:-pair nopair pair}; do
  if [ $v = pair ]; then export VECATTN_PAIR=1; else unset VECATTN_PAIR; fi
  timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --alpha 1.0039 ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$v.json 2> gpurun_out/bench_${TAG}_$v.err
  python - "$v" "gpurun_out/bench_${TAG}_$v.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], {k: d.get(k) for k in ["ms_per_step", "dense_ms", "speedup_vs_dense", "stage_ms", "sparse_achieved_tflops"]}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
