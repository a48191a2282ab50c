#!/bin/bash
# VF_TRACE_SCHEDULE: parity tests, A/B on the headline formats, block timelines with the schedule
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_schedule.py -x -q -p no:cacheprovider > gpurun_out/s_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/s_tests.log)"
timeout 900 python tools/sched_ab.py cfg4 cfg2 cfg3 cfg5 t512 > gpurun_out/s_ab.txt 2>&1; echo "ab rc=$?"
timeout 600 python tools/sched_ab.py cfg4 cfg5 --restart > gpurun_out/s_ab_restart.txt 2>&1; echo "ab restart rc=$?"
for c in cfg2 cfg4 cfg5; do
  VF_LIB=build/variant_clk/libvf.so timeout 300 python tools/block_timeline.py --config $c --schedule > gpurun_out/s_blk_$c.txt 2>&1
  echo "blk $c rc=$?"
done
cat gpurun_out/s_ab.txt gpurun_out/s_ab_restart.txt | grep -v Warn
grep -v Warn gpurun_out/s_blk_*.txt
