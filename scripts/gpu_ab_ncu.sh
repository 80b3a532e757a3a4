#!/bin/bash
bash scripts/gpu_ab.sh
OSPLAT_LIB=$PWD/abtest/lib_a.so TESTS="tests/test_gpu_parity.py tests/test_gpu_loss.py" bash scripts/gpu_tests.sh
for k in k_backward_pixels k_blend k_emit; do
  OSPLAT_LIB=$PWD/abtest/lib_${NCU_VARIANT:-b}.so STEPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${k}_${NCU_VARIANT:-b} python scripts/profile_step.py > /dev/null 2>&1; echo "$k rc=$?"
done
