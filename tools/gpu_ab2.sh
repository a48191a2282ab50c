#!/bin/bash
# A/B of variant libs (build/variant_k5*): python tools/ab_env.py per config
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=""
for v in ${VARIANTS}; do M="$M $v=VF_LIB=build/variant_$v/libvf.so"; done
for spec in ${SPECS:-cfg5: cfg4:}; do
  timeout 1200 python tools/ab_env.py "$spec" $M 2>&1
done
