"""fp32 first-step direction parity of the fused throughput path (B >= 148 -> one chunk,
k_srbd_bwd_fold + k_srbd_fwd_ls) vs the fp64 oracle, over horizons.  Test infrastructure."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from workloads import synth
from tests.gpu_util import rel, rounded, to_device, to_np
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
B = 160
for N in (50, 100, 200, 400, 1000):
    prob = rounded(synth.srbd_problem(B, N=N, seed=N + 1), torch.float32)
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"])
    d = to_device({k: prob[k] for k in ITER}, torch.float32); dirn = h.new_direction()
    h.step(d, direction=dirn); torch.cuda.synchronize()
    errs = []
    for b in range(0, B, 16):
        _, _, _, st, dx, du, dl = O.srbd_step_single(prob, b)
        errs.append(max(rel(to_np(dirn["dx"][b]), dx), rel(to_np(dirn["du"][b]), du), rel(to_np(dirn["dlam"][b]), dl)))
    print(N, "fused fp32 max rel direction err %.2e  median %.2e" % (max(errs), np.median(errs)), flush=True)
