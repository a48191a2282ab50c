#!/bin/bash
# Regenerate the round's GPU evidence on the box (one gpurun call): launch list of the default bench,
# one `ncu --set full` capture of the cfg4 trace kernel, per-format DRAM traffic + instruction counts
# (profiles/traffic.json inputs) and the per-config bench JSON lines. Summaries are written on the
# CPU side with tools/summarize_*.py, tools/traffic_json.py and tools/sweep_table.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFGS=${CFGS:-"cfg4 cfg2 cfg3 cfg5 cfg4i t512 cfg1"}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/full_cfg4 \
  python tools/prof_trace.py --reps 2 > gpurun_out/full_cfg4.log 2>&1
echo "full capture rc=$?"
for c in $CFGS; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum \
    --clock-control none -k regex:trace_ --csv --log-file gpurun_out/traffic_$c.csv \
    python tools/sweep_trace.py $c > gpurun_out/traffic_$c.out 2> gpurun_out/traffic_$c.err
  echo "traffic $c rc=$?"
done
for c in $CFGS; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$? $(head -c 150 gpurun_out/bench_$c.json)"
done
