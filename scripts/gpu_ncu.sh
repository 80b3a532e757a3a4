#!/bin/bash
# GPU box: ncu launch list of a few train steps + full captures of the heavy kernels.
mkdir -p gpurun_out
export STEPS=${STEPS:-3}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
for k in ${KERNELS:-k_blend k_backward_pixels}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k python scripts/profile_step.py > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out
