#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in "$@"; do
  echo "=== case $c"
  timeout 60 python scripts/debug_sparse.py $c 2>&1 | tail -8
  echo "rc=$?"
done
