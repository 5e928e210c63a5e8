mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_dist.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --pre-steps 10 --no-cpu-baseline > gpurun_out/bench_n2_gloo.log 2>&1
cat gpurun_out/pytest_dist.log; tail -3 gpurun_out/bench_n2_gloo.log | cut -c1-600
