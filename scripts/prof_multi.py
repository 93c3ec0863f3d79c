"""One multi-robot SQP step on config 4 (16 robots, n = m = 192, N = 50, B = 1), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
B = int(os.environ.get("MULTI_B", "1"))
p = synth.multi_srbd_problem(B, 16, N=50)
keys = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
it = {k: torch.from_numpy(np.ascontiguousarray(p[k] if p[k].dtype == np.uint8 else p[k].astype(np.float32))).cuda() for k in keys}
h = P.PdIlqr(N=50, n=192, m=192, batch=B, model="multi_srbd", srbd=p["params"], multi=p["multi"])
st = h.step(it)
st = h.step(it, st)
torch.cuda.synchronize()
print("info", st["info"].tolist())
