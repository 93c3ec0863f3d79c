# One GPU call: bench line, ncu launch list of the same command, ncu --set full summaries of the
# fused SRBD kernels (config 3), the latency kernels (B = 1, N = 50) and the large-path fold.
# Outputs: gpurun_out/{bench.log,launches.csv,*_ncu.md,*_ncu.json}
set -x
mkdir -p gpurun_out /tmp/ncu
TAG=${TAG:-r1_v7}
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -c 400 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --latency '' --closed-loop-ticks 0 --no-large > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_srbd_bwd_fold|k_srbd_fwd_ls|k_srbd_lin_rec' -s 3 -c 3 \
  -o /tmp/ncu/fused -f python bench.py --profile-only --steps 3 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/fused.ncu-rep gpurun_out/${TAG}_fused_ncu
LAT_N=50 LAT_CHUNK=1 timeout 600 ncu --set full --clock-control none -k regex:'k_srbd|k_scan|k_policy|k_tail|k_finalize' -s 7 -c 7 \
  -o /tmp/ncu/lat -f python scripts/lat_breakdown.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/lat.ncu-rep gpurun_out/${TAG}_latency_ncu
BIG_CFG=5 BIG_B=1024 timeout 600 ncu --set full --clock-control none -k regex:'k_big' -s 3 -c 3 \
  -o /tmp/ncu/big5 -f python scripts/prof_big.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/big5.ncu-rep gpurun_out/${TAG}_big5_ncu
BIG_CFG=4 BIG_B=1 timeout 600 ncu --set full --clock-control none -k regex:'k_big' -s 3 -c 3 \
  -o /tmp/ncu/big4 -f python scripts/prof_big.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/big4.ncu-rep gpurun_out/${TAG}_big4_ncu
ls -la gpurun_out
