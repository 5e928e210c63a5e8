set -x
mkdir -p gpurun_out; rm -f gpurun_out/bench_face_*
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "quartertile or default or expansion or golden or e64_three" --timeout 600 > gpurun_out/pytest_face.log 2>&1
tail -n 3 gpurun_out/pytest_face.log
for v in 27 27; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --variant $v >> gpurun_out/bench_face_v$v.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_face_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r.get("kernel_ms_avg"), r.get("face_ms_avg"), r["frac"], d["e2e"]["value"], d["ms_per_step"])
PY
