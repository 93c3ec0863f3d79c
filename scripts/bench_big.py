"""Timing of pdilqr_solve_lq on the large-dimension configs (4: n=m=192, N=50, B=1/64;
5: n=74, m=32, N=100, B=1024).  Data: 8 seeded instances tiled over the batch (the algorithm's
work is data-independent)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P

def run(name, B, N, n, m, kind, dtype=torch.float32, reps=5):
    base = synth.random_lq(min(B, 8), N, n, m, kind=kind, seed=7)
    qp = {}
    for k, v in base.items():
        t = torch.from_numpy(v.astype(np.float32 if dtype == torch.float32 else np.float64)).cuda()
        rep = (B + t.shape[0] - 1) // t.shape[0]
        qp[k] = t.repeat((rep,) + (1,) * (t.dim() - 1))[:B].contiguous()
    h = P.PdIlqr(N=N, n=n, m=m, batch=B, dtype=dtype)
    out = h.solve_lq(qp)
    torch.cuda.synchronize()
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): h.solve_lq(qp, out=out)
    e1.record(); torch.cuda.synchronize()
    pr = h.profile_read(); h.profile(False)
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"config": name, "B": B, "N": N, "n": n, "m": m, "dtype": str(dtype), "ms_per_solve_lq": round(ms, 3),
                      "solves_per_s": round(B / ms * 1e3, 1), "kernels_ms": {k: round(v[1] / v[0], 3) for k, v in pr.items()},
                      "info_ok": bool((out["info"] == 0).all())}), flush=True)
    del h

run("config5", 1024, 100, 74, 32, "wb")
run("config4", 1, 50, 192, 192, "dense")
run("config4", 64, 50, 192, 192, "dense")
