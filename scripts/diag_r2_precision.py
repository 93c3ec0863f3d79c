"""Round-2 precision diagnostics (GPU): per-instance fp32 direction errors vs the fp64 oracle, the
KKT backward error eta of the GPU direction on the oracle's QP, and cond(KKT) of a few instances,
for (a) the random-multiplier stress batch (B=64, latency regime), (b) config 3 sampled at B=4096,
(c) config 2 at B=3 / c=1."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O
from tests import kkt_dense
from tests.gpu_util import rel, rounded, to_device, to_np
from workloads import synth
import paper_2506_07823_b200 as P

KEYS = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")


def run(B, N, seed, perturb, idx, leaf_chunk=0, cond_for=()):
    prob = synth.srbd_problem(B, N=N, seed=seed)
    if perturb:
        rng = np.random.default_rng(seed)
        prob["x"] += perturb * rng.standard_normal(prob["x"].shape) * 0.01
        prob["u"] += perturb * rng.standard_normal(prob["u"].shape)
        prob["lam"] += perturb * rng.standard_normal(prob["lam"].shape)
    prob = rounded(prob, torch.float32)
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"], leaf_chunk=leaf_chunk)
    dev = to_device({k: prob[k] for k in KEYS}, torch.float32)
    d = h.new_direction()
    rp = dict(prob)
    h.step(dev, direction=d)
    torch.cuda.synchronize()
    lin = O.srbd_linearize(rp)
    rows = []
    for b in idx:
        _, _, _, st, dx, du, dl = O.srbd_step_single(rp, b)
        e = {k: rel(to_np(d[k][b]), r) for k, r in (("dx", dx), ("du", du), ("dlam", dl))}
        e["eta_gpu"] = kkt_dense.backward_error_blockwise(lin, b, to_np(d["dx"][b]), to_np(d["du"][b]), to_np(d["dlam"][b]))
        e["eta_oracle"] = kkt_dense.backward_error_blockwise(lin, b, dx, du, dl)
        if b in cond_for:
            M, _, _ = kkt_dense.assemble(lin, b)
            e["cond_kkt"] = float(np.linalg.cond(M))
        rows.append((int(b), e))
    return rows


out = {}
out["stress_b64"] = run(64, 50, 32, 1.0, range(64), cond_for=(0, 1, 2, 3))
out["config2_c1"] = run(3, 50, 31, 0.0, range(3), leaf_chunk=1, cond_for=(0,))
idx = [0, 1, 2047, 4095] + list(np.random.default_rng(1).choice(4096, 12, replace=False))
out["config3_b4096"] = run(4096, 50, 34, 0.0, idx, cond_for=(0, 1))
for k, rows in out.items():
    w = {q: max(r[q] for _, r in rows) for q in ("dx", "du", "dlam", "eta_gpu", "eta_oracle")}
    c = [r["cond_kkt"] for _, r in rows if "cond_kkt" in r]
    print(k, "worst", {q: f"{v:.2e}" for q, v in w.items()}, "cond", [f"{v:.2e}" for v in c])
json.dump(out, open("gpurun_out/diag_r2_precision.json", "w"), indent=1, default=float)
