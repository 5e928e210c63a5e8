set -x
mkdir -p gpurun_out
for c in c1 c3 c3_static c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg_$c.log 2>&1
  tail -n 1 gpurun_out/bench_cfg_$c.log | cut -c1-220
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.log 2>&1
tail -n 2 gpurun_out/bench_n2.log | cut -c1-300
