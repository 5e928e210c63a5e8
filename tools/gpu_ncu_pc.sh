# Full ncu capture of one developed-mesh k_main_pc launch (C2 bench workload)
# with source, plus the multi-GPU tests.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_mg.log 2>&1
tail -n 5 gpurun_out/pytest_mg.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_pc --launch-skip 103 -c 1 \
  -o gpurun_out/kpc_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_kpc.log 2>&1
tail -n 3 gpurun_out/ncu_kpc.log
du -sh gpurun_out/kpc_full.ncu-rep
