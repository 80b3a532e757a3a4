#!/bin/bash
# GPU box: A/B of abtest/lib_{VARIANTS}.so including the render sweep (uniform / pole / seam).
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-a b}; do
  OSPLAT_LIB=$PWD/abtest/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/abs_$v.json 2> gpurun_out/abs_$v.err
  python3 -c "import json; d=json.load(open('gpurun_out/abs_$v.json')); r=d['render']; print('$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['kernels_ms_per_step'].items() if k in ('blend','bwd_pixels')}, 'render', round(r['ms_per_frame'],3), {k: round(x['fps_median'],1) for k,x in r['sweep'].items()})"
done
done
