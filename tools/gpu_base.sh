# Session baseline: full GPU parity suite, default bench line, phase probe.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
PLBM_GPU_LIB=build/exp/libphases.so timeout 600 python tools/phase_probe.py > gpurun_out/phases.txt 2>&1
cat gpurun_out/phases.txt
