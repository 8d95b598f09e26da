cp abl/pb2.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py -m gpu -q -x 2>&1 | tail -2
python tools/ab.py "" 3 abl/pb1.so abl/pb2.so
python tools/ab.py "--config c2" 3 abl/pb1.so abl/pb2.so
python tools/ab.py "--config c4 --steps 5" 2 abl/pb1.so abl/pb2.so
