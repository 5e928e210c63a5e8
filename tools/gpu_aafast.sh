set -x
mkdir -p gpurun_out
PLBM_GPU_LIB=build/exp/lib_aafast.so timeout 600 python -m pytest tests -m gpu -q -k "aa and mpmc_e32" 2>&1 | tail -3
PLBM_GPU_LIB=build/exp/lib_aafast.so timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_main_pc --launch-skip 110 -c 2 --csv --log-file gpurun_out/aafast_metrics.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --storage aa > /dev/null 2>&1
