mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 200 gpurun_out/bench.log
cp paper_2506_07823_b200/libpdilqr_ks2.so paper_2506_07823_b200/libpdilqr.so
timeout 900 python -m pytest tests/test_gpu_lq.py tests/test_gpu_srbd.py -q -x > gpurun_out/ks_tests.log 2>&1; tail -4 gpurun_out/ks_tests.log
for ks in 1 0; do PDILQR_KS_SPLIT=$ks LAT_N=25,50,100,1000 LAT_CHUNK=1 timeout 300 python scripts/lat_breakdown.py; done > gpurun_out/lat_ks.log 2>&1; cat gpurun_out/lat_ks.log | cut -c1-300
