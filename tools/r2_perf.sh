python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -n 3 gpurun_out/gpu_tests.log
for a in "" "--kv-heads 1" "--config c2" "--kv-heads 2" "--kv-heads 4"; do
timeout 300 python bench.py $a --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-variant 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%-16s %.4f ms  %.1f steps/s  frac %.3f  passA %.4f' % ('$a', l['ms_per_step'], l['value'], l['hbm_frac_step'], l['roofline']['pass_a_ms']))"
done
python tools/trace.py > gpurun_out/trace_c3.txt 2>&1; python tools/trace.py --kv-heads 1 > gpurun_out/trace_kv1.txt 2>&1; cat gpurun_out/trace_c3.txt gpurun_out/trace_kv1.txt
