#!/bin/bash
# A/B of variant libraries (build/variant_<name>/libvf.so), alternating, two repetitions:
# tools/gpu_ab_var.sh "head vsel" "cfg5 cfg4 t512 cfg2"
cd "$(dirname "$0")/.."
for rep in 1 2; do
for v in $1; do
  for c in $2; do
    echo "$v $(VF_LIB=build/variant_$v/libvf.so timeout 600 python tools/ab_env.py $c: 'base=' 2>&1 | grep -v Warn | head -1)"
  done
done
done
