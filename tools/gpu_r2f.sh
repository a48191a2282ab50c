#!/bin/bash
# bench lines of every config with VF_TRACE_SCHEDULE (index-order value inside each line) and the
# launch list of the default bench's timed step (trace + schedule kernels only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 t512 cfg4s cfg4i; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-side > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.err
  echo "bench $c rc=$?"; cut -c 1-200 gpurun_out/f_bench_$c.json
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"trace_kernel|sched_" --csv \
  --log-file gpurun_out/f_launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-side \
  > gpurun_out/f_launches.log 2>&1
echo "launch list rc=$?"
