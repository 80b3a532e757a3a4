#!/bin/bash
# GPU box: parity tests of the in-tree build (TESTS=...), then the A/B bench of abtest/lib_{VARIANTS}.so.
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/pytest_ab.log
fi
VARIANTS=${VARIANTS:-a b} bash scripts/gpu_ab.sh
