# Full ncu capture of one developed-mesh k_main_pc launch (C2 bench workload),
# exported on the box (the .ncu-rep itself exceeds gpurun's 64 MiB return).
set -x
mkdir -p gpurun_out
LIB=${PLBM_GPU_LIB:-}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_pc --launch-skip 103 -c 1 \
  -o /tmp/kpc_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_kpc.log 2>&1
tail -n 3 gpurun_out/ncu_kpc.log
ncu -i /tmp/kpc_full.ncu-rep --page details --csv > gpurun_out/kpc_details.csv 2>&1
ncu -i /tmp/kpc_full.ncu-rep --page raw --csv > gpurun_out/kpc_raw.csv 2>&1
ncu -i /tmp/kpc_full.ncu-rep --page source --csv --print-source sass > gpurun_out/kpc_sass.csv 2>&1
ncu -i /tmp/kpc_full.ncu-rep --page source --csv --print-source cuda > gpurun_out/kpc_src.csv 2>&1
gzip -f gpurun_out/kpc_sass.csv gpurun_out/kpc_src.csv gpurun_out/kpc_raw.csv
du -sh gpurun_out/*
