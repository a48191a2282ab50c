#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/cnt_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/cnt_tests.log)"; grep -E "^FAILED|Error" gpurun_out/cnt_tests.log | head -10
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:trace_ --csv --log-file gpurun_out/count_launches.csv \
  python tools/prof_trace.py --config cfg5 --counters --reps 1 > gpurun_out/count_launches.log 2>&1
echo "count launches rc=$?"; grep -o '"[^"]*trace_kernel[^"]*"' gpurun_out/count_launches.csv | sort | uniq -c | cut -c1-220
