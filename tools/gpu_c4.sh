mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
timeout 1500 python tools/sweep.py c4 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err
tail -3 gpurun_out/pytest_gpu.log; cut -c1-1500 gpurun_out/sweep_c4.jsonl; tail -3 gpurun_out/sweep_c4.err
