"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
def dev(d, dt=torch.float32):
    return {k: torch.from_numpy(np.ascontiguousarray(v if v.dtype == np.uint8 else v.astype(np.float32 if dt == torch.float32 else np.float64))).cuda()
            for k, v in d.items() if isinstance(v, np.ndarray)}
for (B, N, chunk) in ((3, 9, 0), (3, 9, 1), (2, 9, 4), (150, 6, 0), (150, 6, 1)):
    prob = synth.srbd_problem(B, N=N, seed=1)
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, model="srbd", srbd=prob["params"], leaf_chunk=chunk)
    it = dev({k: prob[k] for k in ITER}); h.step(it); h.linearize(it)
os.environ["PDILQR_SCAN_KS"] = "0"  # latency regime with the Blelloch tree (Kogge-Stone above)
prob = synth.srbd_problem(2, N=9, seed=1)
h = P.PdIlqr(N=9, n=12, m=12, batch=2, model="srbd", srbd=prob["params"], leaf_chunk=1)
h.step(dev({k: prob[k] for k in ITER}))
os.environ.pop("PDILQR_SCAN_KS")
# large path: clusters of 16 / 4 CTAs per instance (B = 1, 3 ... via B) and one CTA per instance (B = 80)
for (n, m, N, chunk, B) in ((5, 3, 7, 0, 3), (12, 12, 7, 3, 3), (4, 2, 5, 1, 3), (20, 9, 4, 0, 3), (20, 9, 4, 0, 1),
                            (20, 9, 3, 0, 80), (40, 36, 2, 0, 2)):
    qp = synth.random_lq(B, N, n, m, seed=2)
    h = P.PdIlqr(N=N, n=n, m=m, batch=B, leaf_chunk=chunk)
    h.solve_lq(dev(qp), policy=True)
torch.cuda.synchronize()
print("sanitize smoke done")
