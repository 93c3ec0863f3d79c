#!/bin/bash
mkdir -p gpurun_out /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_elem_init' -s 1 -c 1 -o /tmp/ncu/elem -f python scripts/prof_lq_only.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/elem.ncu-rep gpurun_out/r2_elem_ncu
ncu -i /tmp/ncu/elem.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_elem_init' > /tmp/ncu/elem_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/elem_src.csv 30 > gpurun_out/r2_elem_lines.txt 2>&1
