#!/bin/bash
# GPU box: one source-correlated ncu capture of kernel $K per library variant (abtest/lib_<v>.so).
mkdir -p gpurun_out
for v in ${VARIANTS:-a b}; do
  OSPLAT_LIB=$PWD/abtest/lib_$v.so STEPS=3 timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"^${K:-k_blend}" -s 2 -c 1 -o gpurun_out/var_${v}_${K:-k_blend} python scripts/profile_step.py \
      > gpurun_out/ncu_var_$v.log 2>&1
  echo "$v rc=$?"
done
