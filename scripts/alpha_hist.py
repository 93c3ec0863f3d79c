"""Histogram of the accepted step size alpha over the first SQP steps of config 3 (B = 4096, N = 50)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
B, N = 4096, 50
prob = synth.srbd_problem(B, N=N, seed=synth.BASE_SEED)
keys = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(np.float32))).cuda() for k in keys}
h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"])
st = h.new_stats()
for s in range(8):
    h.step(it, st)
    torch.cuda.synchronize()
    a = st["alpha"].cpu().numpy()
    print(s, dict(sorted(collections.Counter(np.round(a, 6).tolist()).items(), reverse=True)), flush=True)
