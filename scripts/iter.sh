#!/bin/bash
# Quick GPU iteration: build, GPU parity tests, kernel-only bench line, CTA-0 timeline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; tail -3 gpurun_out/tests.log
timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --alpha 1.0039 ${BENCH_ARGS} > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ["ms_per_step", "forward_ms", "dense_ms", "speedup_vs_dense", "breakdown_two_call", "sparse_achieved_tflops"]}, d["clocks"])
PY
if [ -n "$TRACE" ]; then timeout -s KILL 120 python scripts/trace_run.py video > gpurun_out/trace.log 2>&1; tail -12 gpurun_out/trace.log; fi
