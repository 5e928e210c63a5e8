set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_v0.log 2>&1
timeout 600 python bench.py --variant 1 --no-cpu-baseline > gpurun_out/bench_v1.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --pre-steps 100 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
tail -3 gpurun_out/*.log
