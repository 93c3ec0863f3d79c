"""Timing of pdilqr_solve_lq on the config-3 SRBD linearisation (generic LQ handle, B = 4096, N = 50)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
B, N = 4096, 50
prob = synth.srbd_problem(B, N=N, seed=synth.BASE_SEED)
keys = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(np.float32))).cuda() for k in keys}
hs = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"])
qp = hs.linearize(it); qp.pop("info", None)
h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32)
out = h.solve_lq(qp)
for _ in range(3): h.solve_lq(qp, out=out)
torch.cuda.synchronize()
h.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30): h.solve_lq(qp, out=out)
e1.record(); torch.cuda.synchronize()
pr = h.profile_read()
print(json.dumps({"ms_per_solve_lq": round(e0.elapsed_time(e1) / 30, 4), "kernels_ms": {k: round(v[1] / v[0], 4) for k, v in pr.items()},
                  "info_ok": bool((out["info"] == 0).all())}))
