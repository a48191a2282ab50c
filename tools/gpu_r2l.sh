#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export VF_LIB=build/variant_iters/libvf.so
for r in 1 0; do
  echo "== VF_SCHED_RAYS=$r"
  VF_SCHED_RAYS=$r timeout 900 python tools/sched_ab.py cfg4 cfg5 --reps 9 2>&1 | grep -v Warn
  VF_SCHED_RAYS=$r ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sched_|trace_kernel" --csv --log-file gpurun_out/l_sched_$r.csv \
    python tools/prof_trace.py --config cfg5 --reps 3 --schedule > /dev/null 2>&1
  python tools/summarize_launches.py gpurun_out/l_sched_$r.csv
done
