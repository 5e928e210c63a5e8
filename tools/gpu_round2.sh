# Round-2 evidence: GPU parity (full suite incl. BASELINE-scale goldens),
# smoke, default bench line, the reference arm on the same workload.
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -rA 2>&1 | grep -v "^PASSED" | tail -n 40 > gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref.log 2>&1
tail -n 3 gpurun_out/bench.log gpurun_out/bench_ref.log
