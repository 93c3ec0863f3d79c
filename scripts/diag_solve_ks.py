"""Per-iteration theta / step size of re-solving from a converged iterate (B=6, N=20, fp64) with the
Kogge-Stone and Blelloch latency scans."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
from tests.test_gpu_solve import dev_iter
for ks in ("1", "0"):
    os.environ["PDILQR_SCAN_KS"] = ks
    pr = synth.srbd_problem(6, 20, seed=7)
    h = P.PdIlqr(N=20, n=12, m=12, batch=6, dtype=torch.float64, model="srbd", srbd=pr["params"])
    it = dev_iter(pr, torch.float64)
    st, iters, run = h.solve(it, 50, 1e-9)
    print("ks", ks, "first solve iters", iters.cpu().numpy().tolist())
    for k in range(5):
        d = h.new_direction()
        xs = it["x"].clone(); us = it["u"].clone()
        st = h.step(it, direction=d)
        torch.cuda.synchronize()
        print(f"  step {k}: theta {st['theta'].cpu().numpy()} alpha {st['alpha'].cpu().numpy()} |dx| {d['dx'].abs().amax(dim=(1,2)).cpu().numpy()} |du| {d['du'].abs().amax(dim=(1,2)).cpu().numpy()} info {st['info'].cpu().numpy()}")
