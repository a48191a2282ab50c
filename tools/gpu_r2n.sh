#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do
for v in iters nomov; do
  echo "== $v"
  VF_LIB=build/variant_$v/libvf.so timeout 600 python tools/ab_env.py cfg5: 'base=' 2>&1 | grep -v Warn | head -1
  VF_LIB=build/variant_$v/libvf.so timeout 600 python tools/ab_env.py cfg4: 'base=' 2>&1 | grep -v Warn | head -1
done
done
