python tools/ab.py "--config c3host --steps 8" 2 abl/bc1.so abl/dh1.so
python tools/ab.py "--config c4 --steps 5" 2 abl/bc1.so abl/dh1.so
cp abl/dh1.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
