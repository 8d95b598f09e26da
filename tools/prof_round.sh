# Round evidence: default bench line, launch list of the same command, one --set full capture
# of every step kernel, clocks during the bench.
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
CLK=$!
python bench.py > gpurun_out/bench_$TAG.log 2>&1
kill $CLK
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pass_a|k_select|k_lru_fast|k_pass_b|k_combine|k_dense$|k_group_flags|k_resolve" -s 16 -c 8 -o gpurun_out/full_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
