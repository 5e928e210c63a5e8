set -x
mkdir -p gpurun_out
PLBM_GPU_LIB=build/exp/libphases.so timeout 600 python tools/phase_probe.py 22 > gpurun_out/phases22.txt 2>&1
PLBM_GPU_LIB=build/exp/libphases.so timeout 600 python tools/phase_probe.py 0 > gpurun_out/phases0.txt 2>&1
cat gpurun_out/phases22.txt gpurun_out/phases0.txt
