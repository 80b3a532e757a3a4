#!/bin/bash
# GPU box: parity tests then the default bench line.
mkdir -p gpurun_out
TESTS=${TESTS:-tests} bash scripts/gpu_tests.sh
bash scripts/gpu_bench.sh
