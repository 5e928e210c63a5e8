# ncu evidence for the fused kernel: launch list of the timed steps + one full capture.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 40 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_tm --launch-skip 100 -c 1 \
  -o gpurun_out/tm_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
