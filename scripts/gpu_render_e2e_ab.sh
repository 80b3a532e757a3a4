#!/bin/bash
# GPU box: osplat_render (reference C ABI, host H x W x 3 doubles) FPS for abtest/lib_{VARIANTS}.so.
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-a b}; do
  OSPLAT_LIB=$PWD/abtest/lib_$v.so timeout 600 python scripts/render_e2e_probe.py > gpurun_out/e2e_$v.json 2> gpurun_out/e2e_$v.err
  echo "$v $(tail -1 gpurun_out/e2e_$v.json)"
done
done
