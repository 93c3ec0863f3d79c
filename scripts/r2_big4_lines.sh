#!/bin/bash
# source-line view of k_big_ric at config 4, B = 1 (SIMT products)
mkdir -p gpurun_out /tmp/ncu
BIG_CFG=4 BIG_B=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big_ric' -s 1 -c 1 \
  -o /tmp/ncu/big4 -f python scripts/prof_big.py > /dev/null 2>&1
ncu -i /tmp/ncu/big4.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_big_ric' > /tmp/ncu/big4_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/big4_src.csv 50 > gpurun_out/r2_big4_lines.txt 2>&1
BIG_CFG=5 BIG_B=296 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big_ric' -s 1 -c 1 \
  -o /tmp/ncu/big5 -f python scripts/prof_big.py > /dev/null 2>&1
ncu -i /tmp/ncu/big5.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_big_ric' > /tmp/ncu/big5_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/big5_src.csv 50 > gpurun_out/r2_big5_lines.txt 2>&1
cp /tmp/ncu/big4_src.csv /tmp/ncu/big5_src.csv gpurun_out/
