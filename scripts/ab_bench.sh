#!/bin/bash
# same-box A/B: quick bench of each ab/lib_*.so, interleaved twice
cd "$(dirname "$0")/.."
for rep in 1 2; do for l in ab/lib_*.so; do echo "== $l"; CI_LIB=$PWD/$l bash scripts/quick_bench.sh --inflight 1 "$@"; done; done
