# per-config ncu traffic table + default bench (with the reference cpu_baseline) + reference arm
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python tools/traffic.py c3 c2 c5 c3host c4 > gpurun_out/traffic.log 2>&1; tail -n 6 gpurun_out/traffic.log
cp gpurun_out/traffic_r02.json profiles/traffic_r02.json 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1; tail -n 1 gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; tail -n 1 gpurun_out/bench_ref.log
