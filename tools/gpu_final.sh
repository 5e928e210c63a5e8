# Round evidence: smoke, full GPU suite, default bench line, reference arm on
# the same workload, ncu launch list of the timed steps.
set -x
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -n 2 gpurun_out/smoke.log
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
timeout 1200 python bench.py --impl reference --steps 30 --warmup 5 > gpurun_out/bench_ref.log 2>&1
tail -n 1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 60 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
tail -n 3 gpurun_out/launches.csv
