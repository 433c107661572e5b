#!/bin/bash
# TOPK per-kernel A/B of prebuilt library variants: abtopk.sh tag1 tag2 ...  (main = the in-tree build)
cd "$(dirname "$0")/.."
cp paper_2603_29494_b200/libvecattn.so /tmp/lib_main.so
for v in "$@"; do
  if [ "$v" = main ]; then cp /tmp/lib_main.so paper_2603_29494_b200/libvecattn.so; else cp paper_2603_29494_b200/build/ab/lib_$v.so paper_2603_29494_b200/libvecattn.so; fi
  echo "== $v"; timeout -s KILL 300 python scripts/topk_prof.py 2>&1 | tail -14
done
cp /tmp/lib_main.so paper_2603_29494_b200/libvecattn.so
