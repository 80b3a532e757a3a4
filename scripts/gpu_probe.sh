#!/bin/bash
# GPU box: e2e probe + source-level ncu captures of the two pixel kernels.
mkdir -p gpurun_out
timeout 300 python scripts/e2e_probe.py 2>&1 | tee gpurun_out/e2e_probe.log
for k in ${KERNELS:-k_blend k_backward_pixels}; do
  STEPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 2 -c 1 \
      -o gpurun_out/prof_$k python scripts/profile_step.py > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
