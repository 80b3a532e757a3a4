#!/bin/bash
# GPU box: C5 training speed and the e2e probe for several library builds (abtest/lib_*.so).
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  echo "== $v"
  OSPLAT_LIB=$PWD/abtest/lib_$v.so timeout 600 python scripts/roam_train.py --iterations ${ROAM_ITERS:-5000} 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('roam it/s', round(d['iterations_per_s'],1), 'final', d['final_gaussians'])"
  [ -n "$E2E" ] && OSPLAT_LIB=$PWD/abtest/lib_$v.so timeout 300 python scripts/e2e_probe.py 2>&1 | tail -5
done
