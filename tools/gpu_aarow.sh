set -x
mkdir -p gpurun_out
PLBM_GPU_LIB=build/exp/lib_aarow.so timeout 900 python -m pytest tests -m gpu -q -k "aa and (e32 or c2_100)" > gpurun_out/pytest_aarow.log 2>&1
tail -n 2 gpurun_out/pytest_aarow.log
CAND=aarow BENCH_ARGS="--storage aa" bash tools/gpu_ab_bench.sh
