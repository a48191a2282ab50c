#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_schedule.py tests/test_bench_contract.py -x -q -p no:cacheprovider > gpurun_out/m_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/m_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/m_tests.log | head -8
timeout 900 python tools/sched_ab.py cfg4 cfg5 cfg3 t512 cfg2 --reps 9 2>&1 | grep -v Warn
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sched_|trace_kernel" --csv --log-file gpurun_out/m_sched.csv \
    python -c "
import sys; sys.argv=['x','--config','cfg5','--reps','3']
import torch
exec(open('tools/prof_trace.py').read().replace('schedule=a.schedule','schedule=\"regroup\"'))" > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/m_sched.csv
