# ncu of the E = 64 cluster kernel on C5 (512^3 static, E = 64, C = 2): one
# full capture (exported on the box) + the bench line
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --extent 64 --components 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_e64.log 2>&1
tail -n 1 gpurun_out/bench_c5_e64.log | cut -c1-600
timeout 900 ncu --set full --clock-control none -k regex:k_main_pc --launch-skip 4 -c 1 \
  -o /tmp/e64_full -f python bench.py --config c5 --extent 64 --components 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_e64.log 2>&1
tail -n 2 gpurun_out/ncu_e64.log
ncu -i /tmp/e64_full.ncu-rep --page details --csv > gpurun_out/e64_details.csv 2>&1
ncu -i /tmp/e64_full.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active > gpurun_out/e64_raw.csv 2>&1
du -sh gpurun_out/e64_*
