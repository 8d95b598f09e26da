set -x
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_v3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pass_a|k_pass_b|k_select|k_dense$|k_union" -s 20 -c 6 -o gpurun_out/full_r01_v3 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_full.log 2>&1
ls -la gpurun_out
