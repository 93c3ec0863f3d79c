mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/multi_tests.log 2>&1; tail -25 gpurun_out/multi_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency '' --closed-loop-ticks 0 --no-scan-legs --no-e2e > gpurun_out/bench_large.log 2>&1
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_large.log') if l.startswith('{')][-1])
for k,v in d['large'].items(): print(k, {a:(round(b,3) if isinstance(b,float) else b) for a,b in v.items() if a!='kernels_ms'}, {a: round(b,3) for a,b in v['kernels_ms'].items()})
PY
