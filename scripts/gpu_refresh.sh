#!/bin/bash
# one-box refresh of everything profiles/ quotes (round tag $1, default r02)
cd "$(dirname "$0")/.."
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --config C3R --no-alt --no-extras --cpu-groups 4 --reps 0 > gpurun_out/bench_c3r.json 2> gpurun_out/bench_c3r.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# launch list of the timed configuration (cold-cache, serialised: compare shares)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --inflight 1 --no-e2e --no-alt --no-extras --no-cpu-baseline --reps 0 > /dev/null 2>&1
# full capture of the main-forward stage launches (s0, s1, s2) of the second serve call
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 9 -c 3 -o gpurun_out/prof_stage_$TAG -f \
  python bench.py --steps 1 --warmup 1 --inflight 1 --no-e2e --no-alt --no-extras --no-cpu-baseline --reps 0 > gpurun_out/ncu_full.log 2>&1
# DRAM counters of the HBM-bound kernels (standalone 8192-group launches of the bench's hbm item)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"k_mean|k_decode" --csv --log-file gpurun_out/hbm_dram.csv \
  python bench.py --steps 1 --warmup 1 --inflight 1 --no-e2e --no-alt --no-cpu-baseline --reps 0 > /dev/null 2>&1
# learned-encoder launch list at k = 2, 4, 10 (E1, tail, E4)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/enc_launches.csv \
  python scripts/enc_launches.py > /dev/null 2>&1
python - <<'PY'
import json
for f in ("bench", "bench_c3r", "bench_ref"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"),
          (d.get("numerics") or {}).get("pass"))
PY
