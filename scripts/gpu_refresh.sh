#!/bin/bash
# one-box refresh of everything the profiles/ summary quotes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --cpu-groups 96 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 300 python bench.py --precision fp32 --no-alt --no-cpu-baseline > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
timeout 300 python bench.py --config C4 --no-alt --cpu-groups 8 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config C3R --no-alt --cpu-groups 4 > gpurun_out/bench_c3r.json 2> gpurun_out/bench_c3r.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --inflight 1 --no-e2e --no-alt --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 9 -c 3 -o gpurun_out/prof_stage_r01 \
  python bench.py --steps 1 --warmup 2 --inflight 1 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
for f in bf16 fp32 c4 c3r ref; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
