set -x
mkdir -p gpurun_out; rm -f gpurun_out/bench_q_*
PLBM_BARRIER_TIMEOUT_S=60 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_q_default.log 2>&1
PLBM_FACE_VARIANT=1 timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_q_face1.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_q_default.log 2>&1
PLBM_FACE_VARIANT=1 timeout 600 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_q_face1.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 --storage aa >> gpurun_out/bench_q_aa.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_q_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, d["value"], r.get("kernel_ms_avg"), r.get("face_ms_avg"), r["frac"], d["e2e"]["value"], d["ms_per_step"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_q.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_pc --launch-skip 103 -c 1 \
  -o /tmp/kpc_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_kpc.log 2>&1
ncu -i /tmp/kpc_full.ncu-rep --page details --csv > gpurun_out/kpc_details.csv 2>&1
ncu -i /tmp/kpc_full.ncu-rep --page raw --csv > gpurun_out/kpc_raw.csv 2>&1
gzip -f gpurun_out/kpc_raw.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_face --launch-skip 103 -c 1 \
  -o /tmp/kface_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_kface.log 2>&1
ncu -i /tmp/kface_full.ncu-rep --page details --csv > gpurun_out/kface_details.csv 2>&1
ncu -i /tmp/kface_full.ncu-rep --page source --csv --print-source cuda > gpurun_out/kface_src.csv 2>&1
gzip -f gpurun_out/kface_src.csv
du -sh gpurun_out/*
