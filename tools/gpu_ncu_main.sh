mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_pc --launch-skip 100 -c 1 \
  -o gpurun_out/main_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_main.log 2>&1
du -sh gpurun_out/*
