#!/bin/bash
# A/B of attention variants (kernel table of tools/dbg_refine.py); usage: tools/attn_ab.sh out.txt cfg "env1" "env2" ...
out=$1; cfg=$2; shift 2
for env in "$@"; do
  echo "== $cfg $env" >> $out
  env $env python tools/dbg_refine.py $cfg 2>&1 | grep -E "attention|combine|Error|error" >> $out
done
