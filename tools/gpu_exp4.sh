set -x
mkdir -p gpurun_out
PLBM_BARRIER_TIMEOUT_S=20 timeout 600 python tools/dbg_mg.py mpmc3_static mpmc_e32_solid_periodic mpmc_e64 c1_progressive > gpurun_out/dbg_mg.txt 2>&1
cat gpurun_out/dbg_mg.txt
PLBM_BARRIER_TIMEOUT_S=30 timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_mg.log 2>&1
tail -n 25 gpurun_out/pytest_mg.log
