set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
PLBM_BARRIER_TIMEOUT_S=120 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 --pre-steps 20 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_n2_gloo.log 2>&1
tail -n 3 gpurun_out/bench_n2_gloo.log
