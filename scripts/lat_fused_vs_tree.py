"""B = 1 SQP step latency (CUDA-graph replay, device time) vs horizon: the default latency path
(leaf_chunk = 1: Kogge-Stone scans, 6 kernels) against the fused single-chunk path (leaf_chunk = N+2:
records + sequential fold + rollout/line search, 3 kernels)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
KEYS = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
stream = torch.cuda.Stream()
for N in (25, 50, 100, 200, 400, 1000):
    row = {"N": N}
    for name, lc in (("tree", 1), ("fused", N + 2)):
        prob = synth.srbd_problem(1, N=N, seed=synth.BASE_SEED + 2, randomize=False)
        h = P.PdIlqr(N=N, n=12, m=12, batch=1, dtype=torch.float32, model="srbd", srbd=prob["params"], leaf_chunk=lc)
        it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(np.float32))).cuda() for k in KEYS}
        st = h.new_stats()
        pristine = {k: it[k].clone() for k in ("x", "u", "lam")}
        with torch.cuda.stream(stream):
            for _ in range(3): h.step(it, st, stream=stream)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                h.step(it, st, stream=stream)
            for _ in range(30): g.replay()
            stream.synchronize()
            ts = []
            for _ in range(300):
                for k in ("x", "u", "lam"): it[k].copy_(pristine[k])
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream); g.replay(); e1.record(stream); e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
        row[name + "_p50_us"] = round(float(np.median(ts)), 1)
        row[name + "_launches"] = h.last_launch_count()
        del h, g
    print(json.dumps(row), flush=True)
