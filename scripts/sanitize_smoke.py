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
# tensor-core products of the large-n fold (tcgen05, 3xTF32), one cluster and one CTA per instance
os.environ["PDILQR_BIG_TC"] = "1"
for (n, m, N, B) in ((40, 36, 2, 2), (74, 32, 3, 3)):
    qp = synth.random_lq(B, N, n, m, seed=3)
    P.PdIlqr(N=N, n=n, m=m, batch=B).solve_lq(dev(qp))
os.environ.pop("PDILQR_BIG_TC")
# multi-robot step (R = 2), LQ adjoint, horizon-sharding segment kernels
mp = synth.multi_srbd_problem(2, 2, N=4, seed=1, spacing=0.8)
h = P.PdIlqr(N=4, n=24, m=24, batch=2, model="multi_srbd", srbd=mp["params"], multi=mp["multi"])
h.step(dev({k: mp[k] for k in ITER}))
qp = dev(synth.random_lq(2, 6, 8, 4, seed=4))
h = P.PdIlqr(N=6, n=8, m=4, batch=2)
sol = h.solve_lq(qp)
h.solve_lq_adjoint(qp, sol, {"dx": torch.ones_like(sol["dx"])})
S = h.segment_reduce(qp)
Pe, pe = h.segment_suffix(torch.stack([S, S]), 0, qp["P_term"], qp["p_term"])
F = h.segment_forward(qp)
h.segment_prefix(torch.stack([F, F]), 1, qp["dx0"])
torch.cuda.synchronize()
print("sanitize smoke done")
