#!/bin/bash
# large-n tree scan (leaf_chunk = 1): parity tests and timing at configs 4 (B = 1) and 5 (B = 64)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big_scan.py -q -x 2>&1 | tail -4
timeout 600 python - <<'PY' 2>&1 | tee gpurun_out/bigscan_time.txt
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from workloads import synth
import paper_2506_07823_b200 as P
for name, B, N, n, m, kind in (("config4", 1, 50, 192, 192, "dense"), ("config5", 64, 100, 74, 32, "wb")):
    base = synth.random_lq(min(B, 4), N, n, m, kind=kind, seed=7)
    qp = {}
    for k, v in base.items():
        t = torch.from_numpy(v.astype(np.float32)).cuda()
        rep = (B + t.shape[0] - 1) // t.shape[0]
        qp[k] = t.repeat((rep,) + (1,) * (t.dim() - 1))[:B].contiguous()
    for lc in (0, 1):
        h = P.PdIlqr(N=N, n=n, m=m, batch=B, dtype=torch.float32, leaf_chunk=lc)
        out = h.solve_lq(qp); torch.cuda.synchronize()
        h.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.solve_lq(qp, out=out); e1.record(); torch.cuda.synchronize()
        pr = h.profile_read()
        print(json.dumps({"config": name, "B": B, "leaf_chunk": lc, "ms": round(e0.elapsed_time(e1), 3),
                          "kernels_ms": {k: round(v[1], 3) for k, v in pr.items()}, "info_ok": bool((out["info"] == 0).all())}), flush=True)
        del h
PY
