#!/bin/bash
# ncu evidence for profiles/: launch list of a bench run + --set full of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-r01}
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python scripts/prof_run.py --reps 2 > gpurun_out/launches_$TAG.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 2 \
  -o gpurun_out/prof_attn_$TAG -f python scripts/prof_run.py --reps 2 > gpurun_out/prof_attn_$TAG.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:select_kernel -s 1 -c 1 \
  -o gpurun_out/prof_select_$TAG -f python scripts/prof_run.py --reps 2 --no-dense > gpurun_out/prof_select_$TAG.log 2>&1
ls -la gpurun_out
