mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py c1 > gpurun_out/sweep_c1.jsonl 2> gpurun_out/sweep_c1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --pre-steps 10 --no-cpu-baseline > gpurun_out/bench_n2_gloo.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/sweep_c1.jsonl; tail -2 gpurun_out/sweep_c1.err; tail -1 gpurun_out/bench_n2_gloo.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('exchange'))"
