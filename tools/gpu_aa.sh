set -x
mkdir -p gpurun_out
PLBM_BARRIER_TIMEOUT_S=60 timeout 1200 python -m pytest tests -m gpu -q -x -k "aa" > gpurun_out/pytest_aa.log 2>&1
tail -n 3 gpurun_out/pytest_aa.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 --storage aa > gpurun_out/bench_aa.log 2>&1
tail -n 1 gpurun_out/bench_aa.log | cut -c1-200
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_aa.log").read().strip().splitlines()[-1]); r = d["roofline"]
print("AA", d["value"], r["kernel_ms_avg"], r["frac"], r["face_ms_avg"])
PY
