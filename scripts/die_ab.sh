#!/bin/bash
# A/B of the item scheduler's die split (VECATTN_DIE_SPLIT=0/1/2) on the kernel-level timings.
cd "$(dirname "$0")/.."
for i in 1 2; do for m in 0 1 2; do
  echo "die_mode=$m $(VECATTN_DIE_SPLIT=$m timeout -s KILL 300 python scripts/attn_ab.py ${AB_ARGS} 2>&1 | tail -1)"
done; done
