#!/bin/bash
cd "$(dirname "$0")/.."
VF_LIB=build/variant_k5top/libvf.so python tools/ab_check.py cfg5 cfg4 2>&1 | tail -2
for spec in cfg5: cfg4: t512: "cfg5:R(4, 4, 4) G(8)" "cfg4:R(6, 6, 6) G(5)"; do
  timeout 900 python tools/ab_env.py "$spec" "base=VF_LIB=build/variant_k5base2/libvf.so" "top=VF_LIB=build/variant_k5top/libvf.so" 2>&1
done
