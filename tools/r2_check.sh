# verification suites + api tests on the GPU, then the default bench line (c3 + c3host variant)
export CKV_PARITY_LOG=gpurun_out/parity_report.txt; rm -f $CKV_PARITY_LOG
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_verification_suites.py tests/test_gpu_api.py -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; tail -n 15 gpurun_out/gpu_tests.log
grep verify $CKV_PARITY_LOG
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1; tail -n 3 gpurun_out/bench_c3.log
