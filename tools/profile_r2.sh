#!/bin/bash
# Round-2 GPU evidence (one gpurun call): launch list of the default bench (cfg5), one
# `ncu --set full` capture of the headline trace kernel (+ L1/L2 byte metrics), per-format DRAM
# traffic + instruction counts for profiles/traffic.json, and the cfg4 capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_cfg5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-side > gpurun_out/r2_launches_bench.log 2>&1
echo "launch list rc=$?"
X=lts__t_bytes.sum,l1tex__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum
for c in ${FULL_CFGS:-cfg5 cfg4}; do
  ncu --set full --metrics $X --import-source on --clock-control none -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/r2_full_$c \
    python tools/prof_trace.py --config $c --reps 2 > gpurun_out/r2_full_$c.log 2>&1
  echo "full capture $c rc=$?"
done
for c in ${CFGS:-cfg5 cfg4}; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum \
    --clock-control none -k regex:trace_ --csv --log-file gpurun_out/traffic_$c.csv \
    python tools/sweep_trace.py $c > gpurun_out/traffic_$c.out 2> gpurun_out/traffic_$c.err
  echo "traffic $c rc=$?"
done
