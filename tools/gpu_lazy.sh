set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lazy or eager or halves or expansion_paths" > gpurun_out/pytest_lazy.log 2>&1
tail -n 3 gpurun_out/pytest_lazy.log
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py c4 --steps 400 > gpurun_out/sweep_c4_ab_lazy.jsonl 2>&1
PLBM_LAZY_POOL=0 timeout 900 python tools/sweep.py c4 --steps 400 > gpurun_out/sweep_c4_ab_eager.jsonl 2>&1
timeout 900 python tools/sweep.py c3 --steps 400 > gpurun_out/sweep_c3_lazy.jsonl 2>&1
timeout 300 python bench.py > gpurun_out/bench_lazy.json 2> gpurun_out/bench_lazy.err
python - <<'PY'
import json
for f in ["gpurun_out/sweep_c4_ab_lazy.jsonl", "gpurun_out/sweep_c4_ab_eager.jsonl", "gpurun_out/sweep_c3_lazy.jsonl"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    for k in ("progressive", "static"):
        if k in d:
            print(f, k, d[k]["total_ms"], d[k]["final_tiles"], d[k].get("pool_mapped_GB"), [s["ms"] for s in d[k]["series"]][:8])
PY
cat gpurun_out/bench_lazy.json
