"""fp32 vs fp64 first-step direction parity of pdilqr_step at long horizons (B=1, tree path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from workloads import synth
from tests.gpu_util import rel, rounded, to_device, to_np
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
for N in (50, 100, 200, 400, 1000):
    for dt in (torch.float32, torch.float64):
        prob = rounded(synth.srbd_problem(2, N=N, seed=N, randomize=False), dt)
        h = P.PdIlqr(N=N, n=12, m=12, batch=2, dtype=dt, model="srbd", srbd=prob["params"])
        d = to_device({k: prob[k] for k in ITER}, dt); dirn = h.new_direction()
        h.step(d, direction=dirn); torch.cuda.synchronize()
        errs = []
        for b in range(2):
            _, _, _, st, dx, du, dl = O.srbd_step_single(prob, b)
            errs.append(max(rel(to_np(dirn["dx"][b]), dx), rel(to_np(dirn["du"][b]), du), rel(to_np(dirn["dlam"][b]), dl)))
        print(N, dt, "max rel direction err %.2e" % max(errs), flush=True)
