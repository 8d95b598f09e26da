cp abl/dm1.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_sharded.py tests/test_verification_suites.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/ab.py "--kv-heads 1" 3 abl/bc1.so abl/dm1.so
python tools/ab.py "" 2 abl/bc1.so abl/dm1.so
python tools/trace.py --kv-heads 1
