mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_big.py tests/test_gpu_closed_loop.py tests/test_gpu_solve.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/quick_tests.log 2>&1; tail -4 gpurun_out/quick_tests.log
timeout 900 python bench.py --latency '' --closed-loop-ticks 0 --no-scan-legs --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_q.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernels_ms'])
for k,v in d['large'].items(): print(k, round(v.get('ms_per_step', v.get('ms_per_solve_lq')),3), {a: round(b,3) for a,b in v['kernels_ms'].items()})
PY
