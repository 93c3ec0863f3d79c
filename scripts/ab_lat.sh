for r in 1 2; do for v in base new; do
cp paper_2506_07823_b200/libpdilqr_$v.so paper_2506_07823_b200/libpdilqr.so
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --closed-loop-ticks 0 --no-large --latency 25,50,200,1000 > /tmp/lb.log 2>&1
python -c "
import json;d=json.loads(open('/tmp/lb.log').read().strip().splitlines()[-1])
print('$v', {k:(round(v['p50_us'],1),v['launches']) for k,v in d['latency']['per_dtype']['f32'].items()})"
done; done
