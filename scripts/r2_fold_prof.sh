#!/bin/bash
# ncu --set full of the record-fed fold, the linearisation records and the line search; source-line view
TAG=${1:-r2_v11}
mkdir -p gpurun_out /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_srbd_bwd_fold|k_srbd_fwd_ls|k_srbd_lin_rec' -s 3 -c 3 -o /tmp/ncu/fused -f python bench.py --profile-only --steps 3 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/fused.ncu-rep gpurun_out/${TAG}_fused_ncu
ncu -i /tmp/ncu/fused.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_srbd_bwd_fold' > /tmp/ncu/fold_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/fold_src.csv 60 > gpurun_out/${TAG}_fold_lines.txt 2>&1
cp /tmp/ncu/fused.ncu-rep gpurun_out/${TAG}_fused.ncu-rep
