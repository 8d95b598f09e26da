timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -x 2>&1 | tail -2
python tools/ab.py "" 3 abl/base.so abl/pb1.so
python tools/ab.py "--config c2" 3 abl/base.so abl/pb1.so
cp abl/pb1.so paper_2605_20868_b200/libcertkv_b200.so
