#!/bin/bash
# A/B of static vs dynamic batch claiming, 1 and 2 batches in flight (same box)
cd "$(dirname "$0")/.."
for env in "CI_STATIC_BATCHES=1" "CI_DYN=1"; do
  for f in 1 2; do
    env $env timeout 300 python bench.py --no-alt --no-e2e --no-cpu-baseline --inflight $f "$@" 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', d['config']['inflight'], round(d['value']), round(d['ms_per_step'],3), (d.get('roofline') or {}).get('frac'))"
  done
done
