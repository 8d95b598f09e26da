cp abl/ap1.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/ab.py "" 3 abl/pb2.so abl/ap1.so
python tools/ab.py "--kv-heads 1" 3 abl/pb2.so abl/ap1.so
python tools/ab.py "--config c2" 3 abl/pb2.so abl/ap1.so
cp abl/ap1.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
