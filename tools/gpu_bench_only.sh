# A/B bench of fused-kernel variants without the parity suite: bash tools/gpu_bench_only.sh "0 10"
mkdir -p gpurun_out
for v in ${1:-0}; do
  timeout 600 python bench.py --variant $v --no-cpu-baseline --steps 20 > gpurun_out/bench_v$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v$v.log').read().strip().splitlines()[-1]); print('v$v', d['value'], d['roofline']['kernel_ms_avg'], d['roofline']['face_ms_avg'], d['roofline']['frac'])"
done
