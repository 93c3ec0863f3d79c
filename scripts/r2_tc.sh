mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1; tail -15 gpurun_out/tc_tests.log
timeout 600 python -m pytest tests/test_gpu_big.py tests/test_gpu_adjoint.py -q -p no:cacheprovider > gpurun_out/big_tests.log 2>&1; tail -15 gpurun_out/big_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency '' --closed-loop-ticks 0 --no-scan-legs --no-e2e > gpurun_out/bench_large.log 2>&1; tail -c 1500 gpurun_out/bench_large.log
