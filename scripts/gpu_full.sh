#!/bin/bash
# GPU box: parity tests, default bench line, ncu launch list of the bench command's train steps,
# and one `ncu --set full` capture per hot kernel (traffic + stall evidence for profiles/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv | tee gpurun_out/gpu.txt
if [ -z "$SKIP_TESTS" ]; then
  TESTS=${TESTS:-tests} bash scripts/gpu_tests.sh
fi
bash scripts/gpu_bench.sh
# launch list of the bench's train-step path (cold-cache, serialised: shares, not absolutes)
STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
for k in ${KERNELS:-k_backward_pixels k_blend k_ssim_fwd k_ssim_bwd k_backward_gaussians k_adam k_preprocess k_emit k_downsweep k_upsweep}; do
  STEPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 2 -c 1 \
      -o gpurun_out/prof_$k python scripts/profile_step.py > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out
