#!/bin/bash
# A/B over several device-memory layouts (TCG_ALLOC_PAD_KB): ab_base/ vs working tree
for pad in ${PADS:-0 64 1000 5000 17000}; do
 for c in ${AB_CFGS:-cfg2}; do
  (cd ab_base && TCG_ALLOC_PAD_KB=$pad TAG="BASE pad=$pad" python tools/step_timing.py $c)
  TCG_ALLOC_PAD_KB=$pad TAG="NEW  pad=$pad" python tools/step_timing.py $c
 done
done 2>&1 | grep -E "STEP|rror"
