#!/bin/bash
# GPU box: ncu --set full of every K2 kernel of one frame (render #3 of profile_step) -> gpurun_out/k2.ncu-rep
mkdir -p gpurun_out
STEPS=3 timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_(iota|depth_key24|upsweep|scan_counts|downsweep|fix_runs|touch_sums|scan_block_sums|emit_prep|emit|ranges)" \
   -s 40 -c 24 -o gpurun_out/k2 python scripts/profile_step.py > gpurun_out/ncu_k2.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_k2.log
