#!/bin/bash
# A/B bench.py command-line variants on one GPU box: each argument is a quoted flag string.
for a in "$@"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $a > gpurun_out/ab.json 2>gpurun_out/ab.err
  tail -1 gpurun_out/ab.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('[$a]', d['value'], d['e2e']['value'], 'ms', d['ms_per_step'], 'clk', d['clocks']['sm_mhz'], 'dom', d['roofline']['kernel'], d['roofline']['launch_ms'])" || tail -5 gpurun_out/ab.err
done
