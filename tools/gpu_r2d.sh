#!/bin/bash
# VF_TRACE_SCHEDULE evidence: GPU tests, driver bench line, cfg4 bench line, launch list of the
# default bench, ncu --set full of the cfg4 trace kernel in index order vs scheduled, cfg5 scheduled.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/d_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/d_tests.log)"; grep -E "^FAILED|Error" gpurun_out/d_tests.log | head -5
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
echo "bench rc=$?"; cat gpurun_out/d_bench.json
timeout 900 python bench.py --config cfg4 --steps 20 --warmup 5 --no-side > gpurun_out/d_bench_cfg4.json 2> gpurun_out/d_bench_cfg4.err
echo "bench cfg4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/d_launches_cfg5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-side > gpurun_out/d_launches.log 2>&1
echo "launch list rc=$?"
X=lts__t_bytes.sum,l1tex__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in "cfg4 nat" "cfg4 sched" "cfg5 sched"; do
  set -- $v
  ncu --set full --metrics $X --import-source on --clock-control none -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/d_full_$1_$2 \
    python tools/prof_trace.py --config $1 --reps 2 $([ $2 = sched ] && echo --schedule) > gpurun_out/d_full_$1_$2.log 2>&1
  echo "full $1 $2 rc=$?"
done
