#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in head m8; do
  echo "== $v"; VF_LIB=build/variant_$v/libvf.so timeout 600 python tools/sched_ab.py cfg5 cfg4 --reps 11 2>&1 | grep -v Warn | sed 's/, regroup.*//'
done; done
