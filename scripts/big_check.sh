mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_big.py -q -x > gpurun_out/big_tests.log 2>&1; tail -5 gpurun_out/big_tests.log
timeout 300 python scripts/bench_big.py > gpurun_out/bench_big.log 2>&1; cat gpurun_out/bench_big.log | tail -5
