mkdir -p gpurun_out /tmp/ncu
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1; tail -3 gpurun_out/tc_tests.log
timeout 600 python -m pytest tests/test_gpu_big.py -q -p no:cacheprovider > gpurun_out/big_tests.log 2>&1; tail -8 gpurun_out/big_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency '' --closed-loop-ticks 0 --no-scan-legs --no-e2e > gpurun_out/bench_large.log 2>&1
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_large.log') if l.startswith('{')][-1])
for k,v in d['large'].items(): print(k, round(v['ms_per_solve_lq'],3), {a: round(b,3) for a,b in v['kernels_ms'].items()})
PY
PDILQR_BIG_TC=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency '' --closed-loop-ticks 0 --no-scan-legs --no-e2e > gpurun_out/bench_large_simt.log 2>&1
BIG_CFG=4 BIG_B=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big' -s 5 -c 5 -o /tmp/ncu/big4 -f python scripts/prof_big.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/big4.ncu-rep gpurun_out/r2_v2_big4_ncu
ncu -i /tmp/ncu/big4.ncu-rep --page source --csv --print-source cuda,sass -k regex:'k_big_ric' > /tmp/ncu/big4_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/big4_src.csv 30 > gpurun_out/r2_v2_big4_lines.txt 2>&1; head -35 gpurun_out/r2_v2_big4_lines.txt
BIG_CFG=5 BIG_B=1024 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_big_ric' -s 1 -c 1 -o /tmp/ncu/big5 -f python scripts/prof_big.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/big5.ncu-rep gpurun_out/r2_v2_big5_ncu
ncu -i /tmp/ncu/big5.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu/big5_src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/ncu/big5_src.csv 30 > gpurun_out/r2_v2_big5_lines.txt 2>&1; head -35 gpurun_out/r2_v2_big5_lines.txt
