mkdir -p gpurun_out /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_srbd_bwd_fold|k_srbd_fwd_ls' -s 2 -c 2 -o /tmp/ncu/fused -f python bench.py --profile-only --steps 3 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/fused.ncu-rep gpurun_out/r2_v3_fused_ncu
ncu -i /tmp/ncu/fused.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_srbd_bwd_fold' > /tmp/ncu/fold_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/fold_src.csv 45 > gpurun_out/r2_v3_fold_lines.txt 2>&1
ncu -i /tmp/ncu/fused.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_srbd_fwd_ls' > /tmp/ncu/ls_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/ls_src.csv 45 > gpurun_out/r2_v3_ls_lines.txt 2>&1
head -50 gpurun_out/r2_v3_fold_lines.txt; head -30 gpurun_out/r2_v3_ls_lines.txt
