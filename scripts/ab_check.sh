mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_big.py -q -x > gpurun_out/big_tests.log 2>&1; tail -25 gpurun_out/big_tests.log
timeout 300 python scripts/bench_big.py > gpurun_out/bench_big.log 2>&1; cat gpurun_out/bench_big.log | tail -5
LAT_N=25,50,100,200 LAT_CHUNK=1,0 timeout 300 python scripts/lat_breakdown.py > gpurun_out/lat.log 2>&1; cat gpurun_out/lat.log | tail -8
for r in 1 2; do SWEEP_CONFIGS='[{"fold":4,"ls":4}]' timeout 200 python scripts/sweep_step.py; done > gpurun_out/ab_split.log 2>&1
cp paper_2506_07823_b200/libpdilqr_nosplit.so paper_2506_07823_b200/libpdilqr.so
for r in 1 2; do SWEEP_CONFIGS='[{"fold":4,"ls":4}]' timeout 200 python scripts/sweep_step.py; done > gpurun_out/ab_nosplit.log 2>&1
tail -2 gpurun_out/ab_split.log gpurun_out/ab_nosplit.log
