#!/bin/bash
# GPU box: warm-cache ncu launch lists (serialised, --cache-control none) of the train step for the
# A/B library builds abtest/lib_{VARIANTS}.so — per-kernel intrinsic durations without PDL overlap.
mkdir -p gpurun_out
for v in ${VARIANTS:-a b}; do
  OSPLAT_LIB=$PWD/abtest/lib_$v.so STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
      --cache-control none --csv --log-file gpurun_out/launches_$v.csv python scripts/profile_step.py \
      > gpurun_out/launches_$v.log 2>&1
  echo "$v rc=$?"
  python3 scripts/launch_summary.py gpurun_out/launches_$v.csv --steps 3 --json gpurun_out/launches_$v.json > /dev/null
done
