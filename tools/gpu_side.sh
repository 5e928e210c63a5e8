mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "side or default" 2>&1 | tail -3
for sh in 60 90 120 150; do
  PLBM_SIDE_SHARE=$sh timeout 600 python bench.py --variant 24 --no-cpu-baseline --steps 20 > gpurun_out/bench_side$sh.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_side$sh.log').read().strip().splitlines()[-1]); print('share $sh', d['value'], d['roofline']['kernel_ms_avg'])"
done
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_v0.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_v0.log').read().strip().splitlines()[-1]); print('v0', d['value'], d['roofline']['kernel_ms_avg'])"
