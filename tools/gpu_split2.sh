set -x
mkdir -p gpurun_out; rm -f gpurun_out/bench_split2_*
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
for v in 26 27 26 27; do
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --variant $v >> gpurun_out/bench_split2_v$v.log 2>&1
done
timeout 1500 python tools/sweep.py c5 --extents 32 64 --comps 1 2 3 > gpurun_out/sweep_c5_split.jsonl 2>&1
PLBM_SPLIT=2 timeout 1500 python tools/sweep.py c5 --extents 32 64 --comps 1 2 3 > gpurun_out/sweep_c5_split2.jsonl 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_split2_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r.get("kernel_ms_avg"), r.get("face_ms_avg"), r["frac"], d["e2e"]["value"], d["ms_per_step"])
for f in ["gpurun_out/sweep_c5_split.jsonl", "gpurun_out/sweep_c5_split2.jsonl"]:
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); print(f, d["E"], d["C"], d["mlups_per_comp"], d["k_main_ms"], d["k_face_ms"])
PY
