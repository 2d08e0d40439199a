#!/bin/bash
cd "$(dirname "$0")/.."
for l in ab/lib_*.so; do echo "== $l"; CI_LIB=$PWD/$l bash scripts/quick_bench.sh --inflight 1; done
echo "== nobatch static batches"; CI_STATIC_BATCHES=1 CI_LIB=$PWD/ab/lib_nobatch.so bash scripts/quick_bench.sh --inflight 1
