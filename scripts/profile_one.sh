#!/bin/bash
# usage: TAG=x KREGEX=attn_kernel SKIP=2 ARGS="--heads 2" scripts/profile_one.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-attn_kernel} -s ${SKIP:-2} -c ${COUNT:-1} \
  -o gpurun_out/prof_${TAG:-x} -f python scripts/prof_run.py ${ARGS} > gpurun_out/prof_${TAG:-x}.log 2>&1
tail -3 gpurun_out/prof_${TAG:-x}.log
