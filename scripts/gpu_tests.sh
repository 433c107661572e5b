#!/bin/bash
# Run GPU test groups one at a time with hard timeouts; logs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.log | tail -20; }
for k in "${@:-pool scores selection dense sparse capacity degenerate full_selection}"; do
  for kk in $k; do
    echo "=== $kk" | tee -a gpurun_out/tests.log
    timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$kk" --timeout 300 2>&1 | tail -40 | tee -a gpurun_out/tests.log
  done
done
