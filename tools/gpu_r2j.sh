#!/bin/bash
# ray regrouping inside the schedule: parity tests + A/B (VF_SCHED_RAYS=0 = block order only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_schedule.py tests/test_bench_contract.py -x -q -p no:cacheprovider > gpurun_out/j_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/j_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/j_tests.log | head -8
for r in 1 0; do
  echo "== VF_SCHED_RAYS=$r"
  VF_SCHED_RAYS=$r timeout 900 python tools/sched_ab.py cfg4 cfg5 cfg3 t512 cfg2 --reps 9 2>&1 | grep -v Warn
done
