#!/bin/bash
# GPU box: the non-default BASELINE configs with the current build — C4 (3M, 4096x2048, a fixed batch
# of 8 views per step), C5 (roaming scene densified past 1M Gaussians) — and the full-size parity probe.
mkdir -p gpurun_out
timeout 900 python bench.py --gaussians 3000000 --width 4096 --height 2048 --global-views 8 --steps 5 \
    --no-cpu-baseline --no-sweep > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "c4 rc=$?"
timeout 1200 python scripts/roam_train.py --iterations 30000 --init-points 600000 --densify-grad 3e-5 \
    --prune-radius 1e9 > gpurun_out/roam_1m.json 2> gpurun_out/roam_1m.err
echo "roam rc=$?"
timeout 1500 python scripts/fullsize_parity_probe.py > gpurun_out/parity_probe.log 2>&1
echo "parity rc=$?"
