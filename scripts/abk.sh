#!/bin/bash
# Interleaved kernel-level A/B of prebuilt library variants: abk.sh <rounds> tag1 tag2 ... (args to attn_ab.py in AB_ARGS)
cd "$(dirname "$0")/.."
n=$1; shift
cp paper_2603_29494_b200/libvecattn.so /tmp/lib_main.so
for i in $(seq $n); do for v in "$@"; do
  if [ "$v" = main ]; then cp /tmp/lib_main.so paper_2603_29494_b200/libvecattn.so; else cp paper_2603_29494_b200/build/ab/lib_$v.so paper_2603_29494_b200/libvecattn.so; fi
  echo "$v $(timeout -s KILL 300 python scripts/attn_ab.py ${AB_ARGS} 2>&1 | tail -1)"
done; done
cp /tmp/lib_main.so paper_2603_29494_b200/libvecattn.so
