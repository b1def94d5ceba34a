#!/bin/bash
# A/B a runtime knob on one GPU box: runs bench.py once per "NAME=VALUE" argument, printing
# tokens/s, e2e and the attention / per-kernel ms of each run.  Usage: [WL=cfg5] tools/ab_env.sh A=1 A=2 ...
for kv in "$@"; do
  env $kv timeout 300 python bench.py ${WL:+--workload $WL} --steps 20 --warmup 5 --no-cpu-baseline --no-serving > gpurun_out/ab.json 2>/dev/null
  tail -1 gpurun_out/ab.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$kv', d['value'], d['e2e']['value'], 'clk', d['clocks']['sm_mhz'], ' '.join(f'{n}={v[\"ms_per_step\"]}' for n,v in k.items() if v['ms_per_step']>0.1))"
done
