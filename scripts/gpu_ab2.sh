#!/bin/bash
# GPU box: A/B of library builds (abtest/lib_<v>.so) and of the fused single-view step, bench kernel timings.
mkdir -p gpurun_out
run() {  # name, lib, extra env
  env $3 OSPLAT_LIB=$PWD/abtest/lib_$2.so timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-sweep \
      > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err
  python3 -c "import json; d=json.load(open('gpurun_out/ab_$1.json')); print('$1', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'render', round(d['render']['ms_per_frame'],3))"
}
for rep in 1 2; do
  run a_fused$rep a "X=1"
  run b_fused$rep b "X=1"
  run b_unfused$rep b "OSPLAT_UNFUSED_STEP=1"
done
