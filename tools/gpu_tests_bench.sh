# GPU parity suite + default bench line (+ reference arm) + launch list.
# usage: bash tools/gpu_tests_bench.sh [pytest -k expr]
set -x
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
fi
tail -n 30 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -n 3 gpurun_out/bench.log
