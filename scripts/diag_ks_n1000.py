"""Direction of one SRBD step at B = 1, N = 1000 (latency regime) with the Kogge-Stone and Blelloch scans
vs the fp64 oracle; fp32 and fp64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
from oracle import oracle as O
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
for N in (50, 1000):
    prob = synth.srbd_problem(1, N=N, seed=3, randomize=False)
    for dt in (torch.float32, torch.float64):
        npd = np.float32 if dt == torch.float32 else np.float64
        pr = synth.round_to(prob, npd)
        ref = O.srbd_step_single(pr, 0)
        for ks in ("1", "0"):
            os.environ["PDILQR_SCAN_KS"] = ks
            h = P.PdIlqr(N=N, n=12, m=12, batch=1, dtype=dt, model="srbd", srbd=prob["params"], leaf_chunk=1)
            it = {k: torch.from_numpy(np.ascontiguousarray(pr[k] if pr[k].dtype == np.uint8 else pr[k].astype(npd))).cuda() for k in ITER}
            d = h.new_direction()
            st = h.step(it, direction=d)
            torch.cuda.synchronize()
            errs = []
            for g, r in ((d["dx"][0], ref[4]), (d["du"][0], ref[5]), (d["dlam"][0], ref[6])):
                g = g.cpu().numpy().astype(np.float64)
                errs.append(float(np.abs(g - r).max() / max(np.abs(r).max(), 1e-30)))
            print(f"N={N} {dt} ks={ks} info={int(st['info'][0])} alpha={float(st['alpha'][0])} ref_alpha={ref[3][2]} rel_err dx/du/dlam={errs} max|dx|={float(d['dx'].abs().max())}")
