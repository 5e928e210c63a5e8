# Round evidence: default bench line (+ reference arm), ncu launch list of the
# timed steps, the face kernel's full capture.  The fused kernel's full
# capture (with source) is tools/gpu_ncu_main.sh (gpurun copies back <= 64 MiB).
set -x
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 320 -c 60 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_face --launch-skip 100 -c 1 \
  -o gpurun_out/face_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_face.log 2>&1
du -sh gpurun_out/*; tail -n 2 gpurun_out/smoke.log
