#!/bin/bash
# Round-2 evidence, part A: compute-sanitizer (memcheck / initcheck / racecheck / synccheck), the
# launch list of the default bench, ncu --set full of the cfg5 and cfg4 headline kernels (+ L1/L2
# byte metrics), per-format DRAM traffic + instruction counts (profiles/traffic.json inputs).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K="small_formats and 0.03 or noncubic or payload or empty_volume or query or compiled_in or scatter or align"
for tool in memcheck initcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$K" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?"; tail -2 gpurun_out/sanitize_$tool.log
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_cfg5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-side > gpurun_out/r2_launches_bench.log 2>&1
echo "launch list rc=$?"
X=lts__t_bytes.sum,l1tex__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum
for c in cfg5 cfg4 cfg2; do
  ncu --set full --metrics $X --import-source on --clock-control none -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/r2f_$c \
    python tools/prof_trace.py --config $c --reps 2 > gpurun_out/r2f_$c.log 2>&1
  echo "full capture $c rc=$?"
done
for c in cfg5 cfg4 cfg2 cfg3 t512; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum \
    --clock-control none -k regex:trace_ --csv --log-file gpurun_out/traffic_$c.csv \
    python tools/sweep_trace.py $c > gpurun_out/traffic_$c.out 2> gpurun_out/traffic_$c.err
  echo "traffic $c rc=$?"
done
bash tools/gpu_pack.sh
