"""Diagnostic: where does fp32 precision go on SRBD QPs?  (test infra; uses the oracle)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from workloads import synth
from tests.gpu_util import rel_per_instance, rounded, to_device, to_np
import paper_2506_07823_b200 as P

B, N = 64, 50
prob = synth.srbd_problem(B, N=N, seed=32)
rng = np.random.default_rng(32)
prob["x"] += 0.01 * rng.standard_normal(prob["x"].shape)
prob["u"] += rng.standard_normal(prob["u"].shape)
prob["lam"] += rng.standard_normal(prob["lam"].shape)
prob = rounded(prob, np.float32)
lin = O.srbd_linearize(prob)
lin32 = rounded({k: v for k, v in lin.items() if k != "info"}, np.float32)
for chunk in (1, 52):
    for dt in (torch.float32, torch.float64):
        h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=dt, leaf_chunk=chunk)
        out = h.solve_lq(to_device(lin32, dt)); torch.cuda.synchronize()
        ref = O.solve_lq(lin32)
        print("solve_lq on oracle-linearised QP", chunk, dt, {k: float(rel_per_instance(to_np(out[k]), ref[k]).max()) for k in ("dx", "du", "dlam")})
hs = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"])
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
g = hs.linearize(to_device({k: prob[k] for k in ITER}, torch.float32)); torch.cuda.synchronize()
for k in ("A", "Bm", "c", "R", "q", "r", "p_term", "dx0"):
    a = to_np(g[k]); b = lin[k]
    err = np.abs(a - b)
    print("linearize", k, "max abs err", err.max(), "max |ref|", np.abs(b).max(), "max rel-to-entry", float((err / np.maximum(np.abs(b), 1e-30)).max()))
glin = {k: to_np(g[k]) for k in lin32}
h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32)
out = h.solve_lq(to_device(glin, torch.float32)); torch.cuda.synchronize()
ref = O.solve_lq(lin)
print("gpu lin + gpu solve vs oracle", {k: float(rel_per_instance(to_np(out[k]), ref[k]).max()) for k in ("dx", "du", "dlam")})
ref2 = O.solve_lq(glin)
print("oracle solve on gpu lin vs oracle", {k: float(rel_per_instance(ref2[k], ref[k]).max()) for k in ("dx", "du", "dlam")})
