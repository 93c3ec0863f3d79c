# Round-2 measurement call: GPU tests, smoke, default bench line, ncu launch list of the same bench
# command, ncu --set full summaries of the headline, latency, large-path (SIMT and tcgen05) and
# multi-robot kernels.  Outputs under gpurun_out/ with the tag $TAG.
set -x
TAG=${TAG:-r2_v4}
mkdir -p gpurun_out /tmp/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1; tail -3 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -2 gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -c 300 gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --latency '' --closed-loop-ticks 0 --no-large --no-scan-legs --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_srbd_bwd_fold|k_srbd_fwd_ls' -s 2 -c 2 \
  -o /tmp/ncu/fused -f python bench.py --profile-only --steps 3 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/fused.ncu-rep gpurun_out/${TAG}_fused_ncu
LAT_N=50 LAT_CHUNK=1 timeout 600 ncu --set full --clock-control none -k regex:'k_srbd|k_scan|k_policy|k_tail|k_finalize' -s 7 -c 7 \
  -o /tmp/ncu/lat -f python scripts/lat_breakdown.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/lat.ncu-rep gpurun_out/${TAG}_latency_ncu
BIG_CFG=5 BIG_B=1024 timeout 600 ncu --set full --clock-control none -k regex:'k_big' -s 3 -c 3 \
  -o /tmp/ncu/big5 -f python scripts/prof_big.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/big5.ncu-rep gpurun_out/${TAG}_big5_ncu
PDILQR_BIG_TC=1 BIG_CFG=5 BIG_B=1024 timeout 600 ncu --set full --clock-control none -k regex:'k_big_ric' -s 1 -c 1 \
  -o /tmp/ncu/big5tc -f python scripts/prof_big.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/big5tc.ncu-rep gpurun_out/${TAG}_big5tc_ncu
ncu -i /tmp/ncu/big5tc.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:]:
    for k,v in zip(h,r):
        if ('tensor' in k or 'pipe_tc' in k or 'tmem' in k or 'tcgen' in k) and v: print(k, v)
" > gpurun_out/${TAG}_big5tc_tensor_pipe.txt
timeout 600 ncu --set full --clock-control none -k regex:'k_multi|k_big' -s 7 -c 7 \
  -o /tmp/ncu/multi4 -f python scripts/prof_multi.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/multi4.ncu-rep gpurun_out/${TAG}_multi4_ncu
ls -la gpurun_out
