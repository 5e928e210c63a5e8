set -x
mkdir -p gpurun_out
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py c3 --steps 300 > gpurun_out/sweep_c3_lazy.jsonl 2>&1
timeout 900 python tools/sweep.py c4 --steps 400 > gpurun_out/sweep_c4_ab_lazy.jsonl 2>&1
timeout 1200 python tools/sweep.py c4 --storage aa --static --steps 200 > gpurun_out/sweep_c4_aa_lazy.jsonl 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/sweep_c3_lazy.jsonl", "gpurun_out/sweep_c4_ab_lazy.jsonl", "gpurun_out/sweep_c4_aa_lazy.jsonl"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    for k in ("progressive", "static"):
        if k in d:
            print(f, k, d[k]["total_ms"], d[k]["final_tiles"], d[k]["pool_mapped_GB"], d[k]["series"][-1].get("map_ms"), d.get("speedup_progressive_vs_static"))
PY
