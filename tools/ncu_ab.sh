# ncu metric pass over A/B modes of the chunked kernels: bash tools/ncu_ab.sh CFG "mode chunk crefill" ...
L=${VF_AB_LIB:-build/variant_chunk5/libvf.so}
CFG=$1; shift
M=smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__grid_size,sm__cycles_active.avg,smsp__warp_issue_stalled_no_instruction_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_branch_resolving_per_warp_active.pct,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,launch__registers_per_thread,smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct,smsp__warp_issue_stalled_membar_per_warp_active.pct,smsp__warp_issue_stalled_drain_per_warp_active.pct
i=0
for mode in "$@"; do
 set -- $mode
 VF_LIB=$L VF_CHUNKED=$1 VF_CHUNK=$2 VF_CREFILL=$3 ncu --metrics $M --clock-control none -k regex:trace_ -s 2 -c 1 --csv --log-file gpurun_out/ncu_ab_${CFG}_$i.csv python tools/prof_trace.py --config $CFG --reps 3 > /dev/null 2>&1
 echo "$mode" > gpurun_out/ncu_ab_${CFG}_$i.mode
 i=$((i+1))
done
