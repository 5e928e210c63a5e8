set -x
mkdir -p gpurun_out
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_lazy.json 2> gpurun_out/bench_lazy.err
timeout 300 python bench.py --storage aa > gpurun_out/bench_lazy_aa.json 2> gpurun_out/bench_lazy_aa.err
timeout 1200 python tools/sweep.py c4 --storage aa --static --steps 200 > gpurun_out/sweep_c4_aa_lazy.jsonl 2>&1
cat gpurun_out/bench_lazy.json gpurun_out/bench_lazy_aa.json | cut -c1-300
