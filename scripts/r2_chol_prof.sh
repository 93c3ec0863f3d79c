mkdir -p gpurun_out /tmp/ncu
BIG_CFG=4 BIG_B=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big_ric|k_big_rchk' -s 2 -c 2 -o /tmp/ncu/b4 -f python scripts/prof_big.py > /dev/null 2>&1
ncu -i /tmp/ncu/b4.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_big_rchk' > /tmp/ncu/rchk_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/rchk_src.csv 30 > gpurun_out/r2_rchk_lines.txt 2>&1
ncu -i /tmp/ncu/b4.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_big_ric' > /tmp/ncu/ric_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/ric_src.csv 40 > gpurun_out/r2_ric4_lines.txt 2>&1
head -32 gpurun_out/r2_rchk_lines.txt; head -42 gpurun_out/r2_ric4_lines.txt
