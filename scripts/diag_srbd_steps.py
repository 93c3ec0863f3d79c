"""Diagnostic: fp32 direction parity of pdilqr_step on the config-2/3 workload, per step (test infra)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from workloads import synth
from tests.gpu_util import rel_per_instance, rounded, to_device, to_np
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
B, N = 64, 50
for chunk in (52, 8, 1):
    prob = rounded(synth.srbd_problem(B, N=N, seed=7), np.float32)
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"], leaf_chunk=chunk)
    dev = to_device({k: prob[k] for k in ITER}, torch.float32)
    dirn = h.new_direction()
    for s in range(4):
        cur = {k: to_np(dev[k]) for k in ("x", "u", "lam")}
        rp = dict(prob); rp.update(cur)
        st = h.step(dev, direction=dirn); torch.cuda.synchronize()
        errs = {k: [] for k in ("dx", "du", "dlam")}; amis = 0
        for b in range(B):
            x, u, lam, st_r, dx, du, dl = O.srbd_step_single(rp, b)
            for k, ref in (("dx", dx), ("du", du), ("dlam", dl)):
                g = to_np(dirn[k][b]); errs[k].append(np.abs(g - ref).max() / np.abs(ref).max())
            amis += int(to_np(st["alpha"])[b] != st_r[2])
        print("chunk", chunk, "step", s, {k: "%.2e" % max(v) for k, v in errs.items()}, "alpha mismatches", amis,
              "mean alpha", float(to_np(st["alpha"]).mean()), "theta", float(to_np(st["theta"]).mean()))
