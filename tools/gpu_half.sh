set -x
mkdir -p gpurun_out; rm -f gpurun_out/bench_half_*
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "halftile or wholetile or expansion or golden" --timeout 600 > gpurun_out/pytest_half.log 2>&1
tail -n 3 gpurun_out/pytest_half.log
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -x --timeout 800 > gpurun_out/pytest_half_large.log 2>&1
tail -n 3 gpurun_out/pytest_half_large.log
for v in 0 20 0 20; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --variant $v >> gpurun_out/bench_half_v$v.log 2>&1
done
for v in 0 20; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --variant $v --storage aa >> gpurun_out/bench_half_aa_v$v.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_half_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r.get("kernel_ms_avg"), r["frac"], d["e2e"]["value"])
PY
