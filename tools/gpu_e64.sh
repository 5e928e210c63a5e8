# E = 64 on the cluster kernel: parity + C5 sweep
set -x
mkdir -p gpurun_out
PLBM_BARRIER_TIMEOUT_S=30 timeout 1200 python -m pytest tests -m gpu -q -x -k "e64" > gpurun_out/pytest_e64.log 2>&1
tail -n 5 gpurun_out/pytest_e64.log
timeout 1200 python tools/sweep.py c5 > gpurun_out/sweep_c5.jsonl 2>&1
cat gpurun_out/sweep_c5.jsonl
