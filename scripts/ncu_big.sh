mkdir -p gpurun_out /tmp/ncu
C=${BIG_CFG:-5}; B=${BIG_B:-296}
BIG_CFG=$C BIG_B=$B timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_big_ric -s 1 -c 1 -o /tmp/ncu/big$C -f python scripts/prof_big.py > gpurun_out/ncu_big$C.log 2>&1
ncu -i /tmp/ncu/big$C.ncu-rep --page details --csv > gpurun_out/big${C}_details.csv 2>&1
ncu -i /tmp/ncu/big$C.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/big${C}_cs.csv 2>&1
ls -la gpurun_out
