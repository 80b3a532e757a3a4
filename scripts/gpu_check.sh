#!/bin/bash
# GPU box: selected GPU tests (TESTS) + the default bench line and optional extra bench lines
# (BENCH2="args" -> gpurun_out/bench2.json).
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/pytest_check.log
fi
timeout 900 python bench.py --no-cpu-baseline --no-sweep ${BENCH_ARGS} > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err
python3 -c "import json; d=json.load(open('gpurun_out/bench_check.json')); print('default', round(d['ms_per_step'],3), round(d['value'],1), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'e2e', round(d['e2e']['value'],1))"
if [ -n "$BENCH2" ]; then
  timeout 900 python bench.py --no-cpu-baseline --no-sweep $BENCH2 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
  python3 -c "import json; d=json.load(open('gpurun_out/bench2.json')); print('bench2', round(d['ms_per_step'],3), round(d['value'],1), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'e2e', round(d['e2e']['value'],1))"
fi
