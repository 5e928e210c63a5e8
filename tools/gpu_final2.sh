# Round evidence after the split-tile clusters: smoke, bench line, reference
# arm, launch list of developed-mesh steps, the BASELINE config sweeps.
set -x
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -n 2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
timeout 900 python bench.py --storage aa > gpurun_out/bench_aa.log 2>&1
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
tail -n 1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 60 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 python tools/sweep.py c1 > gpurun_out/sweep_c1.jsonl 2>&1
timeout 900 python tools/sweep.py c3 --steps 300 > gpurun_out/sweep_c3.jsonl 2>&1
timeout 900 python tools/sweep.py c3 --steps 300 --storage aa > gpurun_out/sweep_c3_aa.jsonl 2>&1
timeout 1200 python tools/sweep.py c4 --storage aa --static --steps 200 > gpurun_out/sweep_c4_aa.jsonl 2>&1
timeout 1200 python tools/sweep.py c4 --static --steps 200 > gpurun_out/sweep_c4_ab.jsonl 2>&1
timeout 2400 python tools/sweep.py c5 --n 512 --extents 32 64 > gpurun_out/sweep_c5_512.jsonl 2>&1
timeout 900 python tools/sweep.py c5 --extents 16 > gpurun_out/sweep_c5_256_e16.jsonl 2>&1
ls -la gpurun_out
