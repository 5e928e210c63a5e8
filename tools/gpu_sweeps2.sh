mkdir -p gpurun_out
timeout 1500 python tools/sweep.py c3 > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err
timeout 1500 python tools/sweep.py c4 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err
timeout 900 python tools/sweep.py c1 > gpurun_out/sweep_c1.jsonl 2> gpurun_out/sweep_c1.err
python -c "
import json
d=json.load(open('gpurun_out/sweep_c3.jsonl')); print('c3', d['progressive']['total_ms'], d['static']['total_ms'], d['speedup_progressive_vs_static'])
d=json.load(open('gpurun_out/sweep_c4.jsonl')); print('c4', d['total_ms'], d['final_tiles'], d['mlups_per_comp'])
d=json.load(open('gpurun_out/sweep_c1.jsonl')); print('c1', d['gpu_ms'], d['ref_s'], d['speedup'], d['same_log_and_counters'])
"
tail -2 gpurun_out/*.err
