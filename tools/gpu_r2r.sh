#!/bin/bash
cd "$(dirname "$0")/.."
VF_LIB=build/variant_adapt/libvf.so timeout 900 python tools/sched_ab.py cfg5 cfg4 t512 cfg2 --reps 15 2>&1 | grep -v Warn
VF_LIB=build/variant_adapt/libvf.so timeout 900 python -m pytest tests/test_schedule.py -q -x -p no:cacheprovider 2>&1 | tail -2
