set -x
mkdir -p gpurun_out; rm -f gpurun_out/bench_ab_*
for lib in base lag2 late base lag2 late; do
  PLBM_GPU_LIB=build/exp/lib_$lib.so timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_ab_$lib.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_ab_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r["kernel_ms_avg"], r["frac"], d["ms_per_step"])
PY
