#!/bin/bash
# Runs on the GPU box (gpurun): GPU parity tests, logs to gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv | tee gpurun_out/gpu.txt
timeout ${TEST_TIMEOUT:-900} python -m pytest ${TESTS:-tests} -x -q -m gpu ${PYTEST_ARGS} 2>&1 | tail -60 | tee gpurun_out/pytest_gpu.log
