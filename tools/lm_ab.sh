#!/bin/bash
# LM-head timing A/B: tools/lm_ab.sh out.txt
out=$1
for cfg in "cfg2 greedy" "cfg2 sample" "cfg5 greedy" "cfg5 sample"; do
  for env in "X=1" "SPECEDGE_LM_PAIR=1"; do
    echo "== $cfg $env" >> $out
    env $env python tools/dbg_refine.py $cfg 2>&1 | grep -E "lm|rmsnorm|Error|error" >> $out
  done
done
