set -x
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -n 2 gpurun_out/smoke.log
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 2400 python tools/sweep.py c5 --n 512 --extents 32 64 > gpurun_out/sweep_c5_512.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
grep "^{" gpurun_out/sweep_c5_512.jsonl | cut -c1-200
grep "^{" gpurun_out/bench.log | cut -c1-200
