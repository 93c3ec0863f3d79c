mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_srbd.py -q -x -p no:cacheprovider > gpurun_out/srbd_tests.log 2>&1; tail -3 gpurun_out/srbd_tests.log
timeout 900 python bench.py --latency '' --closed-loop-ticks 0 --no-scan-legs --no-cpu-baseline --no-large > gpurun_out/bench_e.log 2>&1
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_e.log') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['e2e'])
PY
