mkdir -p gpurun_out
for ks in 1 0; do
PDILQR_SCAN_KS=$ks LAT_N=1000 LAT_CHUNK=1 timeout 300 ncu --clock-control none -k regex:k_srbd_ls_multi -s 3 -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,lts__t_bytes.sum,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio python scripts/lat_breakdown.py 2>&1 | grep -v "^{" | tail -14
done > gpurun_out/ls_diag.log 2>&1
cat gpurun_out/ls_diag.log
