"""One pdilqr_solve_lq on a large-dimension config, for ncu (env BIG_CFG=5|4, BIG_B)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
cfg = os.environ.get("BIG_CFG", "5")
B = int(os.environ.get("BIG_B", "296"))
N, n, m, kind = (100, 74, 32, "wb") if cfg == "5" else (50, 192, 192, "dense")
base = synth.random_lq(min(B, 4), N, n, m, kind=kind, seed=7)
qp = {}
for k, v in base.items():
    t = torch.from_numpy(v.astype(np.float32)).cuda()
    rep = (B + t.shape[0] - 1) // t.shape[0]
    qp[k] = t.repeat((rep,) + (1,) * (t.dim() - 1))[:B].contiguous()
h = P.PdIlqr(N=N, n=n, m=m, batch=B, dtype=torch.float32)
out = h.solve_lq(qp)
out = h.solve_lq(qp, out=out)
torch.cuda.synchronize()
print("info ok", bool((out["info"] == 0).all()))
