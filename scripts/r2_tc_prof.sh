mkdir -p gpurun_out /tmp/ncu
PDILQR_BIG_TC=1 BIG_CFG=4 BIG_B=64 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big_ric' -s 1 -c 1 -o /tmp/ncu/b4tc -f python scripts/prof_big.py > /dev/null 2>&1
ncu -i /tmp/ncu/b4tc.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu/b4tc_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/b4tc_src.csv 45 > gpurun_out/r2_b4tc_lines.txt 2>&1
python scripts/ncu_summary.py /tmp/ncu/b4tc.ncu-rep gpurun_out/r2_b4tc_ncu
BIG_CFG=4 BIG_B=64 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big_ric' -s 1 -c 1 -o /tmp/ncu/b4s -f python scripts/prof_big.py > /dev/null 2>&1
ncu -i /tmp/ncu/b4s.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu/b4s_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/b4s_src.csv 45 > gpurun_out/r2_b4simt_lines.txt 2>&1
head -48 gpurun_out/r2_b4tc_lines.txt; head -30 gpurun_out/r2_b4simt_lines.txt
