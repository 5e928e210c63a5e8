# ncu metrics of the two A-A step kinds (C2 bench workload, A-A storage)
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_main_pc --launch-skip 110 -c 2 --csv --log-file gpurun_out/aa_metrics.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --storage aa > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_main_pc --launch-skip 110 -c 1 --csv --log-file gpurun_out/ab_metrics.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
