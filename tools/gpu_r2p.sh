#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/reps
X=lts__t_bytes.sum,l1tex__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in "cfg4 2073600" "cfg5 8294400"; do
  set -- $v
  ncu --set full --metrics $X --import-source on --clock-control none -k regex:trace_kernel -s 2 -c 1 -o /tmp/reps/p_$1_regroup \
    python tools/prof_trace.py --config $1 --reps 3 --regroup > gpurun_out/p_$1.log 2>&1
  echo "full $1 rc=$?"
  python tools/summarize_ncu.py /tmp/reps/p_$1_regroup.ncu-rep $2 "$1 scheduled + regrouped (VF_TRACE_REGROUP)" > gpurun_out/p_$1_regroup.md 2>&1
done
