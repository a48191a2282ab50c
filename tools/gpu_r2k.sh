#!/bin/bash
# ray regrouping (lane-exit clock key, 8-bit classes): parity + A/B + order-kernel durations
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_schedule.py -x -q -p no:cacheprovider > gpurun_out/k_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/k_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/k_tests.log | head -8
for r in 1 0; do
  echo "== VF_SCHED_RAYS=$r"
  VF_SCHED_RAYS=$r timeout 900 python tools/sched_ab.py cfg4 cfg5 cfg3 t512 cfg2 --reps 9 2>&1 | grep -v Warn
done
for c in cfg5 cfg2; do
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sched_|trace_kernel" --csv --log-file gpurun_out/k_sched_$c.csv \
  python tools/prof_trace.py --config $c --reps 3 --schedule > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/k_sched_$c.csv
done
