#!/bin/bash
# A/B of GEMM variants (kernel table of tools/dbg_refine.py); usage: tools/gemm_ab.sh out.txt cfg "env1" ...
out=$1; cfg=$2; shift 2
for env in "$@"; do
  echo "== $cfg $env" >> $out
  env $env python tools/dbg_refine.py $cfg 2>&1 | grep -E "gemm|rmsnorm|Error|error" >> $out
done
