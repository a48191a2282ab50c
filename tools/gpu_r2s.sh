#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in head scan; do
  echo "== $v"; VF_LIB=build/variant_$v/libvf.so timeout 600 python tools/sched_ab.py t512 cfg2 cfg4 cfg5 --reps 11 2>&1 | grep -v Warn | sed 's/, moved.*//'
done; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sched_" --csv --log-file /tmp/sc.csv env VF_LIB=build/variant_scan/libvf.so python tools/prof_trace.py --config cfg5 --reps 3 --schedule > /dev/null 2>&1
python tools/summarize_launches.py /tmp/sc.csv
