mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 1200 python tools/sweep.py c5 > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
timeout 1500 python tools/sweep.py c3 > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/sweep_c5.jsonl; tail -3 gpurun_out/sweep_c5.err; cut -c1-600 gpurun_out/sweep_c3.jsonl; tail -3 gpurun_out/sweep_c3.err
