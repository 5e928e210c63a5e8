# A-A bench + C4 static on one GPU (A-A), cluster rank interleave experiment
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_ab.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 20 --storage aa > gpurun_out/bench_aa.log 2>&1
for lib in base il base il; do
  PLBM_GPU_LIB=build/exp/lib_$lib.so timeout 600 python bench.py --no-cpu-baseline --steps 20 >> gpurun_out/bench_il_$lib.log 2>&1
done
PLBM_GPU_LIB=build/exp/lib_base.so timeout 300 python tools/probe_cluster.py > gpurun_out/probe_base.txt 2>&1
PLBM_GPU_LIB=build/exp/lib_il.so timeout 300 python tools/probe_cluster.py > gpurun_out/probe_il.txt 2>&1
PLBM_GPU_LIB=build/exp/lib_il_ph.so timeout 600 python tools/phase_probe.py > gpurun_out/phases_il.txt 2>&1
timeout 1500 python tools/sweep.py c4 --storage aa --static --steps 200 > gpurun_out/sweep_c4_aa.jsonl 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r["kernel_ms_avg"], r["frac"], r["face_ms_avg"], d["e2e"]["value"])
PY
cat gpurun_out/probe_*.txt gpurun_out/phases_il.txt
tail -c 3000 gpurun_out/sweep_c4_aa.jsonl
