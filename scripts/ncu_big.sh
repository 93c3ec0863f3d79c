mkdir -p gpurun_out /tmp/ncu
BIG_CFG=5 BIG_B=296 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_big_ric -s 1 -c 1 -o /tmp/ncu/big5 -f python scripts/prof_big.py > gpurun_out/ncu_big5.log 2>&1
BIG_CFG=4 BIG_B=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_big_ric -s 1 -c 1 -o /tmp/ncu/big4 -f python scripts/prof_big.py > gpurun_out/ncu_big4.log 2>&1
for c in big5 big4; do
  ncu -i /tmp/ncu/$c.ncu-rep --page details --csv > gpurun_out/${c}_details.csv 2>&1
  ncu -i /tmp/ncu/$c.ncu-rep --page source --csv --print-source sass > gpurun_out/${c}_sass.csv 2>&1
  ncu -i /tmp/ncu/$c.ncu-rep --page source --csv --print-source cuda > gpurun_out/${c}_src.csv 2>&1
done
ls -la gpurun_out
