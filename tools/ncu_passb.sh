python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_pass_b" -s 6 -c 1 -o gpurun_out/passb_c3 -f python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pass_b|k_select|k_dense$|k_combine" -s 24 -c 4 -o gpurun_out/tail_kv1 -f python bench.py --kv-heads 1 --steps 3 --warmup 5 --no-cpu-baseline --no-e2e --no-variant > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
