#!/bin/bash
# Runs on the GPU box: default bench line (+ optional extra args), logs to gpurun_out/.
mkdir -p gpurun_out
timeout ${BENCH_TIMEOUT:-900} python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "rc=$?"
tail -5 gpurun_out/bench.err
cat gpurun_out/bench.json
