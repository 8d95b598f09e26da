python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q > gpurun_out/sharded_tests.log 2>&1; tail -n 3 gpurun_out/sharded_tests.log
for N in 2 4; do
CKV_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_onedev_n$N.log 2>&1; tail -n 2 gpurun_out/bench_onedev_n$N.log | cut -c1-600
done
