mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x > gpurun_out/lat_tests.log 2>&1; tail -2 gpurun_out/lat_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --closed-loop-ticks 0 --no-large > gpurun_out/lat_bench.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/lat_bench.log').read().strip().splitlines()[-1])
print({k:(round(v['p50_us'],1),v['launches']) for k,v in d['latency']['per_dtype']['f32'].items()})"
