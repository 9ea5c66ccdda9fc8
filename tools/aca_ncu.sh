# quick ncu metrics of the ACA kernels for several libhmx builds
for lib in "$@"; do
  HMX_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct -k regex:aca_kernel -c 2 python tools/ncu_target.py U32k 1 2>&1 | grep -E "aca_kernel|duration|bytes|pct|per_cycle" | sed "s|^|$(basename $lib) |" | cut -c1-150
done
