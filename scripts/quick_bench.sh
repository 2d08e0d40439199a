#!/bin/bash
# quick device-only bench: throughput + per-stage kernel times (single-stream profiled pass)
cd "$(dirname "$0")/.."
timeout 400 python bench.py --no-alt --no-e2e --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'clk', d['clocks']['sm_mhz'])
for k,v in d.get('kernels',{}).items(): print(' ', k, v)
"
