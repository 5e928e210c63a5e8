# A/B of two experiment builds (E32 C2): parity subset with the candidate, then
# alternating bench runs.  usage: bash tools/gpu_ab.sh <candidate> [<baseline>]
set -x
mkdir -p gpurun_out
CAND=${1:-opt}; BASE=${2:-base}
PLBM_GPU_LIB=build/exp/lib_$CAND.so timeout 900 python -m pytest tests -m gpu -q -x -k "(mpmc_e32 and (default or aa_)) or c2_100 or (blowup and e32)" > gpurun_out/pytest_$CAND.log 2>&1
tail -n 3 gpurun_out/pytest_$CAND.log
for lib in $BASE $CAND $BASE $CAND; do
  PLBM_GPU_LIB=build/exp/lib_$lib.so timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_ab_$lib.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_ab_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r["kernel_ms_avg"], r["frac"], r["face_ms_avg"])
PY
