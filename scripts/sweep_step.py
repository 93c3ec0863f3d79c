"""Timing sweep of pdilqr_step over tuning knobs (env PDILQR_OCC_*, leaf_chunk) on config 3."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
B = int(os.environ.get("SWEEP_B", "4096")); N = int(os.environ.get("SWEEP_N", "50"))
dt = torch.float64 if os.environ.get("SWEEP_DTYPE") == "f64" else torch.float32
prob = synth.srbd_problem(B, N=N, seed=synth.BASE_SEED)
npd = np.float32 if dt == torch.float32 else np.float64
def upload():
    return {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(npd))).cuda() for k in ITER}
configs = json.loads(os.environ.get("SWEEP_CONFIGS", '[{"fold":2,"ls":2,"chunk":0}]'))
for c in configs:
    os.environ["PDILQR_OCC_FOLD"] = str(c.get("fold", 2)); os.environ["PDILQR_OCC_LS"] = str(c.get("ls", 2))
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=dt, model="srbd", srbd=prob["params"], leaf_chunk=c.get("chunk", 0))
    it = upload(); st = h.new_stats()
    for _ in range(5): h.step(it, st)
    torch.cuda.synchronize()
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K = 30
    for _ in range(K): h.step(it, st)
    e1.record(); torch.cuda.synchronize()
    prof = h.profile_read(); h.profile(False)
    ms = e0.elapsed_time(e1) / K
    print(json.dumps({"cfg": c, "ms_per_step": round(ms, 4), "solves_per_s": round(B / ms * 1e3),
                      "kernels_ms": {k: round(v[1] / v[0], 4) for k, v in prof.items()}}), flush=True)
    del h
