set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lazy or eager or halves" > gpurun_out/pytest_lazy.log 2>&1
tail -n 3 gpurun_out/pytest_lazy.log
for g in 64 512; do
PLBM_POOL_GRANULE_MB=$g timeout 900 python tools/sweep.py c3 --steps 300 > gpurun_out/sweep_c3_lazy_g$g.jsonl 2>&1
done
PLBM_LAZY_POOL=0 timeout 900 python tools/sweep.py c3 --steps 300 > gpurun_out/sweep_c3_eager.jsonl 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/sweep_c3_lazy_g64.jsonl", "gpurun_out/sweep_c3_lazy_g512.jsonl", "gpurun_out/sweep_c3_eager.jsonl"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    for k in ("progressive",):
        print(f, k, d[k]["total_ms"], d["static"]["total_ms"], [(s["ms"], s.get("map_ms")) for s in d[k]["series"]])
PY
