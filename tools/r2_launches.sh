# per-kernel launch lists (ncu gpu__time_duration, clock-control none) for the step configs
python -c "import __graft_entry__ as g; g.build()" || exit 1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
ncu $M --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_kv1.csv python bench.py --kv-heads 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_c3x.csv python bench.py --explore 0.02 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
for c in c3 kv1 c3x c2; do python tools/launches.py gpurun_out/launches_$c.csv > gpurun_out/launches_${c}_summary.txt 2>&1; done
timeout 600 python bench.py --kv-heads 1 --steps 20 --warmup 5 --no-cpu-baseline --no-variant > gpurun_out/bench_kv1.log 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
ls gpurun_out
