#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/gpu_r2final.sh
timeout 900 python tools/sched_ab.py t512 cfg2 cfg4 cfg5 --reps 11 2>&1 | grep -v Warn | sed 's/, regroup.*//'
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sched_" --csv --log-file /tmp/sc.csv python tools/prof_trace.py --config cfg5 --reps 3 --schedule > /dev/null 2>&1
python tools/summarize_launches.py /tmp/sc.csv
