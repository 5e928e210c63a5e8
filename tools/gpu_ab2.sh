# quick A/B: parity subset, bench kernel time for variants, phase probe
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "${1:-percomp or default or p5 or blowup or golden}" > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
for v in ${2:-0 22 0 22}; do
  timeout 600 python bench.py --variant $v --no-cpu-baseline --steps 20 >> gpurun_out/bench_ab.log 2>&1
done
PLBM_GPU_LIB=build/exp/libphases.so timeout 600 python tools/phase_probe.py > gpurun_out/phases.txt 2>&1
PLBM_GPU_LIB=build/exp/libphases.so timeout 600 python tools/phase_probe.py 22 > gpurun_out/phases22.txt 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench_ab.log"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(d["value"], r["kernel_ms_avg"], r["frac"], r["face_ms_avg"])
PY
