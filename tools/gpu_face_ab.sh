# A/B of k_face variants (PLBM_FACE_VARIANT 0..3) on the default bench
set -x
mkdir -p gpurun_out
for rep in 1; do
for v in 0 1 2 3; do
  PLBM_FACE_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_face$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_face$v.log').read().strip().splitlines()[-1]); print('face$v', d['value'], d['roofline']['kernel_ms_avg'], d['roofline']['face_ms_avg'])"
done
done
PLBM_FACE_VARIANT=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
