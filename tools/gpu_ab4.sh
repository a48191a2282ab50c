#!/bin/bash
cd "$(dirname "$0")/.."
for spec in "cfg4:S(3) G(8)" "cfg4:S(7) G(4)" "cfg4:R(4, 4, 4) S(3) G(4)" "cfg4:R(1, 1, 1) T(2, 5)" "cfg5:T(2, 6)" "cfg3:T(2, 5)" "cfg2:T(2, 4)" "cfg2:" "cfg3:" "cfg5:" "cfg4:"; do
  timeout 900 python tools/ab_env.py "$spec" "chain=" "nochain=VF_LIB=build/variant_nochain/libvf.so" 2>&1
done
