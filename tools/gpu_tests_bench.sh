# GPU parity suite + default bench line.
# usage: bash tools/gpu_tests_bench.sh [pytest -k expr]
set -x
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  PLBM_BARRIER_TIMEOUT_S=60 timeout 1800 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
fi
tail -n 3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
