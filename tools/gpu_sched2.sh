#!/bin/bash
# VF_TRACE_SCHEDULE policy A/B: class granularity (VF_SCHED_SUB) and neighbour dilation (VF_SCHED_DIL)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pol in "2 0" "0 0" "2 2" "2 6" "1 2"; do
  set -- $pol
  echo "== sub=$1 dil=$2"
  VF_SCHED_SUB=$1 VF_SCHED_DIL=$2 timeout 600 python tools/sched_ab.py cfg4 cfg3 cfg5 t512 cfg2 --reps 9 2>&1 | grep -v Warn
done > gpurun_out/s2_ab.txt
cat gpurun_out/s2_ab.txt
