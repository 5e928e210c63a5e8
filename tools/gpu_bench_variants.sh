# bench-only A/B of fused-kernel variants: bash tools/gpu_bench_variants.sh "0 24"
mkdir -p gpurun_out
for v in ${1:-0}; do
  timeout 600 python bench.py --variant $v --no-cpu-baseline --steps 20 > gpurun_out/bench_v$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v$v.log').read().strip().splitlines()[-1]); r=d['roofline']; print('v$v', d['value'], d['config']['tiles'], r['kernel_ms_avg'], r['achieved'], r['frac'], r['face_ms_avg'])"
done
