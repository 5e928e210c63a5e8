# parity + A/B bench of fused-kernel variants: bash tools/gpu_ab.sh "0 2"
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for v in ${1:-0}; do
  timeout 600 python bench.py --variant $v --no-cpu-baseline --steps 20 > gpurun_out/bench_v$v.log 2>&1
done
tail -n 3 gpurun_out/pytest_gpu.log
for v in ${1:-0}; do python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v$v.log').read().strip().splitlines()[-1]); print('v$v', d['value'], d['roofline']['kernel_ms_avg'], d['roofline']['face_ms_avg'], d['roofline']['frac'])"; done
