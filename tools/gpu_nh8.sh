set -x
mkdir -p gpurun_out
PLBM_GPU_LIB=build/exp/lib_nh8.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "e64 and (default or quartertile or halftile or expansion or three)" --timeout 600 > gpurun_out/pytest_nh8.log 2>&1
tail -n 2 gpurun_out/pytest_nh8.log
PLBM_GPU_LIB=build/exp/lib_nh8.so timeout 1500 python tools/sweep.py c5 --n 512 --extents 64 > gpurun_out/sweep_c5_e64_nh8.jsonl 2>&1
timeout 1500 python tools/sweep.py c5 --n 512 --extents 64 > gpurun_out/sweep_c5_e64_nh4.jsonl 2>&1
PLBM_GPU_LIB=build/exp/lib_nh8.so timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_nh8_c2.log 2>&1
cat gpurun_out/sweep_c5_e64_nh8.jsonl gpurun_out/sweep_c5_e64_nh4.jsonl | grep "^{" | cut -c1-240
grep "^{" gpurun_out/bench_nh8_c2.log | cut -c1-120
