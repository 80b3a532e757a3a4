#!/bin/bash
# GPU box: A/B the bench between two library builds in abtest/ (kernel timings only), twice each.
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-a b}; do
  OSPLAT_LIB=$PWD/abtest/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-sweep ${BENCH_ARGS} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python3 -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'render', round(d['render']['ms_per_frame'],3))"
done
done
