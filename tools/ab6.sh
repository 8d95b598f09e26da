cp abl/bc1.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/ab.py "" 3 abl/ap1.so abl/bc1.so
CKV_PB_CHUNKS=6 python tools/ab.py "" 2 abl/bc1.so
CKV_PB_CHUNKS=4 python tools/ab.py "" 2 abl/bc1.so
python tools/ab.py "--kv-heads 1" 3 abl/ap1.so abl/bc1.so
python tools/ab.py "--config c2" 3 abl/ap1.so abl/bc1.so
CKV_PB_CHUNKS=5 python tools/ab.py "--config c2" 2 abl/bc1.so
