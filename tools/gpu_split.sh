set -x
mkdir -p gpurun_out; rm -f gpurun_out/bench_split_*
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile or expansion or golden or default" --timeout 600 > gpurun_out/pytest_split.log 2>&1
tail -n 3 gpurun_out/pytest_split.log
for v in 20 26 27 20 26 27; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --variant $v >> gpurun_out/bench_split_v$v.log 2>&1
done
for v in 26 27; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --variant $v --storage aa >> gpurun_out/bench_split_aa_v$v.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_split_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r.get("kernel_ms_avg"), r.get("face_ms_avg"), r["frac"], d["e2e"]["value"], d["ms_per_step"])
PY
