#!/bin/bash
# GPU box: full evidence pass for profiles/: parity tests, default bench line, ncu launch list of
# the train step, one ncu --set full capture per hot kernel, the C4 (3M, 4096x2048, 8 views) bench
# line and the C5 roaming-scene training run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv | tee gpurun_out/gpu.txt
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
bash scripts/gpu_bench.sh > gpurun_out/bench_log.txt 2>&1
STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > /dev/null 2>&1
echo "launch list rc=$?"
for spec in ${KERNELS:-"k_backward_pixels 2" "k_blend 2" "k_preprocess 2" "k_adam 2" "k_backward_gaussians 2" "k_ssim_fwd 2" "k_ssim_bwd 2" "k_emit 4" "k_downsweep 10"}; do
  set -- $spec
  STEPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$1" -s $2 -c 1 \
      -o gpurun_out/prof_$1 python scripts/profile_step.py > /dev/null 2>&1
  echo "$1 rc=$?"
done
if [ -z "$SKIP_CONFIGS" ]; then
  timeout 900 python bench.py --gaussians 3000000 --width 4096 --height 2048 --views-per-gpu 8 --steps 5 \
      --no-cpu-baseline --no-sweep > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
  echo "c4 rc=$?"
  timeout 1500 python scripts/roam_train.py --iterations ${ROAM_ITERS:-30000} > gpurun_out/roam.json 2> gpurun_out/roam.err
  echo "roam rc=$?"
fi
ls -la gpurun_out
