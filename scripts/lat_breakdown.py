"""Per-kernel breakdown of one B=1 pdilqr_step (config 2) for a few horizons and leaf chunks."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
ITER = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
for N in [int(v) for v in os.environ.get("LAT_N", "50,1000").split(",")]:
    for chunk in [int(v) for v in os.environ.get("LAT_CHUNK", "1,0").split(",")]:
        c = chunk if chunk > 0 else N + 2
        prob = synth.srbd_problem(1, N=N, seed=3, randomize=False)
        h = P.PdIlqr(N=N, n=12, m=12, batch=1, dtype=torch.float32, model="srbd", srbd=prob["params"], leaf_chunk=c)
        it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(np.float32))).cuda() for k in ITER}
        st = h.new_stats()
        for _ in range(5): h.step(it, st)
        torch.cuda.synchronize(); h.profile(True)
        for _ in range(20): h.step(it, st)
        pr = h.profile_read(); h.profile(False)
        print(json.dumps({"N": N, "chunk": c, "kernels_us": {k: round(v[1] / v[0] * 1e3, 1) for k, v in pr.items()},
                          "sum_us": round(sum(v[1] / v[0] for v in pr.values()) * 1e3, 1)}), flush=True)
