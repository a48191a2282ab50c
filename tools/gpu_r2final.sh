#!/bin/bash
# round-2 final evidence: GPU tests, smoke, driver bench line, launch list of the bench's timed
# steps, ncu --set full of the headline kernel (scheduled) and of cfg4 / cfg2 scheduled
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/reps
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/z_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/z_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/z_tests.log | head -8
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/z_smoke.log)"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
echo "bench rc=$?"; cat gpurun_out/z_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"trace_kernel|sched_" --csv \
  --log-file gpurun_out/z_launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-side \
  > gpurun_out/z_launches.log 2>&1
echo "launch list rc=$?"
X=lts__t_bytes.sum,l1tex__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in "cfg5 8294400" "cfg4 2073600" "cfg2 1048576"; do
  set -- $v
  ncu --set full --metrics $X --import-source on --clock-control none -k regex:trace_kernel -s 2 -c 1 -o /tmp/reps/z_$1 \
    python tools/prof_trace.py --config $1 --reps 3 --schedule > gpurun_out/z_full_$1.log 2>&1
  echo "full $1 rc=$?"
  python tools/summarize_ncu.py /tmp/reps/z_$1.ncu-rep $2 "$1 final round-2 build, VF_TRACE_SCHEDULE (third launch)" > gpurun_out/z_full_$1.md 2>&1
done
