#!/bin/bash
# Runs on the GPU box (via gpurun): GPU parity tests with per-test timeouts, logs under gpurun_out/.
# PYTEST_K: optional -k expression.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
if [ -n "$PYTEST_K" ]; then
  timeout ${GPU_TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout ${GPU_TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest exit: $?" >> gpurun_out/pytest_gpu.log
tail -${TAIL_LINES:-60} gpurun_out/pytest_gpu.log
