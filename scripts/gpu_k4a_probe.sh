#!/bin/bash
# GPU box: K4a loop statistics (instrumented build abtest/lib_stats.so) + one ncu --set full capture
# of K4a with source correlation (read back here with ncu -i ... --page source).
mkdir -p gpurun_out
OSPLAT_LIB=$PWD/abtest/lib_stats.so timeout 600 python scripts/k4a_stats.py > gpurun_out/k4a_stats.json 2> gpurun_out/k4a_stats.err
echo "stats rc=$?"; cat gpurun_out/k4a_stats.json; tail -3 gpurun_out/k4a_stats.err
for k in ${KERNELS:-k_backward_pixels k_blend}; do
  STEPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 2 -c 1 \
      -o gpurun_out/src_$k python scripts/profile_step.py > gpurun_out/ncu_src_$k.log 2>&1
  echo "$k rc=$?"
done
