# Full GPU suite + default bench line
set -x
mkdir -p gpurun_out
PLBM_BARRIER_TIMEOUT_S=30 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
tail -n 30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
