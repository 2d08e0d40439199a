mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --cpu-groups 96 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 300 python bench.py --precision fp32 --no-alt --no-cpu-baseline > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-alt --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 9 -c 3 -o gpurun_out/prof_stage_r01 python bench.py --steps 1 --warmup 2 --no-e2e --no-alt --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/bench_bf16.json gpurun_out/bench_fp32.json; tail -3 gpurun_out/bench_bf16.err
