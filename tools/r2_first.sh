python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_c3.log 2>&1; tail -n 1 gpurun_out/r2a_c3.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --tier2 host --scratch 2048 > gpurun_out/r2a_c3host.log 2>&1; tail -n 3 gpurun_out/r2a_c3host.log
nproc; lscpu | head -20 > gpurun_out/r2a_lscpu.txt; free -g >> gpurun_out/r2a_lscpu.txt
