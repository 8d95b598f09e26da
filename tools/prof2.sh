python -c "import __graft_entry__ as g; g.build()"
TAG=${TAG:-v4}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_pass_a|k_pass_b|k_select|k_dense$|k_combine|k_lru}" -s ${SKIP:-20} -c ${CNT:-8} -o gpurun_out/full_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_full.log 2>&1
