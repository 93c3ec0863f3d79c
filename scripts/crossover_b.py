"""Step time vs batch size B (N = 50, fp32, CUDA-graph replay): tree path (leaf_chunk 1) vs fused
single-chunk path (leaf_chunk N+2) -- where the default schedule should switch (DESIGN D1)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
KEYS = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
N = int(os.environ.get("XN", "50"))
stream = torch.cuda.Stream()
for B in (1, 4, 16, 32, 64, 96, 128, 148, 192, 256, 512):
    row = {"B": B, "N": N}
    for name, lc in (("tree", 1), ("chunk8", 8), ("fused", N + 2)):
        prob = synth.srbd_problem(B, N=N, seed=synth.BASE_SEED)
        h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"], leaf_chunk=lc)
        it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(np.float32))).cuda() for k in KEYS}
        st = h.new_stats()
        pristine = {k: it[k].clone() for k in ("x", "u", "lam")}
        with torch.cuda.stream(stream):
            for _ in range(3): h.step(it, st, stream=stream)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                h.step(it, st, stream=stream)
            for _ in range(10): g.replay()
            stream.synchronize()
            ts = []
            for _ in range(100):
                for k in ("x", "u", "lam"): it[k].copy_(pristine[k])
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream); g.replay(); e1.record(stream); e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
        row[name + "_us"] = round(float(np.median(ts)), 1)
        del h, g
    print(json.dumps(row), flush=True)
