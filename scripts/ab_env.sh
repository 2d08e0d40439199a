#!/bin/bash
# same-library A/B of an environment switch: ab_env.sh VAR=1 [bench args]
cd "$(dirname "$0")/.."
SW="$1"; shift
for rep in 1 2; do
  echo "== default"; bash scripts/quick_bench.sh --inflight 1 "$@"
  echo "== $SW"; env "$SW" bash scripts/quick_bench.sh --inflight 1 "$@"
done
