set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_mg.log 2>&1
tail -n 30 gpurun_out/pytest_mg.log
PLBM_GPU_LIB=build/exp/libphases.so timeout 600 python tools/phase_probe.py 22 > gpurun_out/phases22.txt 2>&1
cat gpurun_out/phases22.txt
