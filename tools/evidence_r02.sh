# Round-2 evidence in one GPU call: the GPU test suite (parity / verification logs),
# smoke, the default bench line (C3 + its c3host / exploration variants), the kv1
# proxy and C2 lines, the reference arm, the per-config ncu DRAM table behind
# roofline.traffic, the launch list of the default command, one `ncu --set full`
# capture of each step kernel, and the step timelines.  Outputs in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
export CKV_PARITY_LOG=gpurun_out/parity_report.txt; rm -f $CKV_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -n 3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_r02_c3.log 2>&1
timeout 600 python bench.py --kv-heads 1 --no-variant > gpurun_out/bench_r02_kv1.log 2>&1
timeout 600 python bench.py --config c2 --no-variant > gpurun_out/bench_r02_c2.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_r02_reference.log 2>&1
timeout 2400 python tools/traffic.py c3 c2 c5 c3host c4 > gpurun_out/traffic.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_r02.csv > gpurun_out/launches_r02_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_kv1.csv python bench.py --kv-heads 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_r02_kv1.csv > gpurun_out/launches_r02_kv1_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_c2.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_r02_c2.csv > gpurun_out/launches_r02_c2_summary.txt
ncu --set full --clock-control none --import-source on -k regex:"k_pass_a|k_select|k_pass_b|k_combine|k_dense$|k_append1|k_publish" -s 28 -c 7 -o gpurun_out/full_r02 -f python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_r02.ncu-rep > gpurun_out/ncu_r02_full_summary.txt
ncu --set full --clock-control none --import-source on -k regex:"k_select|k_pass_b|k_combine|k_dense$" -s 16 -c 4 -o gpurun_out/full_r02_kv1 -f python bench.py --kv-heads 1 --steps 3 --warmup 5 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_r02_kv1.ncu-rep > gpurun_out/ncu_r02_kv1_summary.txt
python tools/trace.py > gpurun_out/trace_r02_c3.txt 2>&1
python tools/trace.py --kv-heads 1 > gpurun_out/trace_r02_kv1.txt 2>&1
python tools/trace.py --ctx 32768 > gpurun_out/trace_r02_c2.txt 2>&1
cat gpurun_out/launches_r02_summary.txt
