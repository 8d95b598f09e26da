python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_explore.py tests/test_gpu_baselines.py -k "explore" -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -n 3 gpurun_out/gpu_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3x.csv python bench.py --explore 0.02 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c3x.csv
timeout 600 python bench.py --explore 0.02 --steps 20 --warmup 5 --no-cpu-baseline --no-variant --no-e2e > gpurun_out/bench_c3x.log 2>&1; tail -n 1 gpurun_out/bench_c3x.log | cut -c1-200
