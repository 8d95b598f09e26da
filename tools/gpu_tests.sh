# GPU loop: build check, pytest -m gpu (optionally a subset), smoke
export CKV_PARITY_LOG=gpurun_out/parity_report.txt; rm -f $CKV_PARITY_LOG
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout ${TEST_TIMEOUT:-1200} python -m pytest ${TESTS:-tests} -m gpu -q ${PYTEST_ARGS:--x} > gpurun_out/gpu_tests.log 2>&1; tail -n 30 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 3 gpurun_out/smoke.log
