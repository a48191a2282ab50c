#!/bin/bash
# tests + traffic of the new cfg5 sweep + ncu captures (headline, A/B pairs) + racecheck subset + bench default
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f1_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/f1_tests.log)"; grep -E "^FAILED|Error" gpurun_out/f1_tests.log | head -10
for c in cfg5 cfg4; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum \
    --clock-control none -k regex:trace_ --csv --log-file gpurun_out/traffic_$c.csv \
    python tools/sweep_trace.py $c > gpurun_out/traffic_$c.out 2> gpurun_out/traffic_$c.err
  echo "traffic $c rc=$?"
done
X=lts__t_bytes.sum,l1tex__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum
ncu --set full --metrics $X --import-source on --clock-control none -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/r2g_cfg5 \
  python tools/prof_trace.py --config cfg5 --reps 2 > gpurun_out/r2g_cfg5.log 2>&1
echo "full cfg5 rc=$?"
M=smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_bytes.sum,lts__t_bytes.sum,dram__bytes_read.sum,l1tex__t_sector_hit_rate.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active
for c in cfg5 cfg4; do
  for al in "" "--align"; do
    ncu --metrics $M --clock-control none -k regex:trace_ -s 1 -c 1 --csv --log-file gpurun_out/ncuab_align_${c}${al}.csv \
      python tools/prof_trace.py --config $c --format "R(4, 4, 4) G($([ $c = cfg5 ] && echo 8 || echo 7))" --reps 2 $al > /dev/null 2>&1
  done
  for mode in 1 2; do
    VF_LIB=build/variant_chunk5/libvf.so VF_CHUNKED=$mode VF_CHUNK=32 VF_CREFILL=32 ncu --metrics $M --clock-control none -k regex:trace_ -s 1 -c 1 --csv \
      --log-file gpurun_out/ncuab_stage_${c}_$mode.csv python tools/prof_trace.py --config $c --format "R(4, 4, 4) G($([ $c = cfg5 ] && echo 8 || echo 7))" --reps 2 > /dev/null 2>&1
  done
done
echo "ncu ab done"
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "compiled_in or scatter or empty_volume or query" > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck exit=$?"; tail -2 gpurun_out/sanitize_racecheck.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; cat gpurun_out/bench_default.json
bash tools/gpu_pack.sh
