# Final round evidence: GPU parity suite, smoke, bench (+reference arm), launch list, face capture.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
bash tools/gpu_evidence.sh
