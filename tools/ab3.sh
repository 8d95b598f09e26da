UNITS=32 timeout 600 python tools/selprof.py 2>&1 | tail -12
rm -f paper_2605_20868_b200/libcertkv_b200_prof.so
cp abl/ds1.so paper_2605_20868_b200/libcertkv_b200.so; touch paper_2605_20868_b200/libcertkv_b200.so
ncu --set full --clock-control none --import-source on -k regex:"k_select|k_pass_b|k_combine|k_dense$" -s 8 -c 4 -o gpurun_out/kv1_full -f python bench.py --kv-heads 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/kv1_full.ncu-rep > gpurun_out/ncu_kv1_summary.txt
python tools/ab.py "--kv-heads 1" 3 abl/pf1.so abl/ds1.so
