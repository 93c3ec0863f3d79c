"""NEXT-2: horizon sharding of one LQ problem over G chunks (include/pdilqr.h pdilqr_lq_segment_*;
paper_2506_07823_b200/horizon.py).  The assembled chunk solutions must equal the fp64 oracle's
solve of the whole horizon (rel <= 1e-9 in fp64, 1e-4 in fp32; KKT backward error), with the G
ranks simulated phase by phase in one process (G = 1..8, ragged chunks) and, through the real
torch.distributed path (torchrun, gloo, two ranks sharing the GPU), with two processes."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from tests import kkt_dense
from tests.gpu_util import rel, rounded, to_np
from workloads import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def simulate(P, qp, G, dtype, leaf_chunk=0):
    """All G ranks of horizon.solve_lq_sharded in one process (the two all-gathers become stacks)."""
    from paper_2506_07823_b200 import horizon
    B, N1, n, _ = qp["A"].shape
    m = qp["Bm"].shape[-1]
    N = N1 - 1
    qpt = {k: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", dtype) for k, v in qp.items()}
    chunks = horizon.split_stages(N, G)
    hs, locs = [], []
    for (s, e) in chunks:
        hs.append(P.PdIlqr(N=e - s - 1, n=n, m=m, batch=B, dtype=dtype, leaf_chunk=leaf_chunk))
        locs.append(horizon.local_problem(qpt, s, e))
    S_all = torch.stack([h.segment_reduce(l) for h, l in zip(hs, locs)])
    outs, F = [], []
    for r, (h, l) in enumerate(zip(hs, locs)):
        Pe, pe = h.segment_suffix(S_all, r, qpt["P_term"], qpt["p_term"])
        l.update(P_term=Pe, p_term=pe, dx0=torch.zeros_like(qpt["dx0"]))
        outs.append(h.solve_lq(l))
        F.append(h.segment_forward(l))
    F_all = torch.stack(F)
    for r, (h, l) in enumerate(zip(hs, locs)):
        l["dx0"] = h.segment_prefix(F_all, r, qpt["dx0"])
        outs[r] = h.solve_lq(l, out=outs[r])
    torch.cuda.synchronize()
    dx = np.concatenate([to_np(o["dx"][:, :-1]) for o in outs] + [to_np(outs[-1]["dx"][:, -1:])], axis=1)
    dl = np.concatenate([to_np(o["dlam"][:, :-1]) for o in outs] + [to_np(outs[-1]["dlam"][:, -1:])], axis=1)
    du = np.concatenate([to_np(o["du"]) for o in outs], axis=1)
    info = np.stack([to_np(o["info"]) for o in outs])
    return dx, du, dl, info


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("G,N,n,m,kind", [(1, 20, 12, 12, "dense"), (2, 40, 12, 12, "dense"), (3, 50, 8, 4, "dense"),
                                          (8, 200, 12, 12, "dense"), (4, 63, 16, 16, "dense"), (5, 30, 6, 2, "wb"),
                                          (2, 1, 4, 2, "dense")])
def test_sharded_equals_whole_horizon(P, O, dtype, G, N, n, m, kind):
    B = 3
    qp = rounded(synth.random_lq(B, N, n, m, seed=N + G, kind=kind), dtype)
    dx, du, dl, info = simulate(P, qp, G, dtype)
    assert (info == 0).all()
    ref = O.solve_lq(qp)
    tol = 1e-9 if dtype == torch.float64 else 1e-4
    for k, v in (("dx", dx), ("du", du), ("dlam", dl)):
        for b in range(B):
            assert rel(v[b], ref[k][b]) <= tol, (k, b, rel(v[b], ref[k][b]))
    for b in range(B):
        assert kkt_dense.backward_error_blockwise(qp, b, dx[b], du[b], dl[b]) <= (1e-12 if dtype == torch.float64 else 1e-5)


def test_srbd_linearisation_long_horizon_sharded(P, O):
    """The paper's use case for horizon parallelism: one SRBD instance with a long horizon (N = 400),
    its LQ subproblem (oracle linearisation) solved in 4 chunks."""
    prob = synth.srbd_problem(1, N=400, seed=9, randomize=False)
    qp = O.srbd_linearize(prob)
    qp.pop("info")
    dx, du, dl, info = simulate(P, qp, 4, torch.float64)
    ref = O.solve_lq(qp)
    assert (info == 0).all()
    for k, v in (("dx", dx), ("du", du), ("dlam", dl)):
        assert rel(v[0], ref[k][0]) <= 1e-8, k


def test_two_processes_gloo(P, O, tmp_path):
    out = str(tmp_path / "h.npz")
    N, n, m, B = 30, 12, 12, 2
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29573",
                        os.path.join(ROOT, "scripts", "horizon_worker.py"), out, str(N), str(n), str(m), str(B), "dense"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    g = np.load(out)
    assert (g["info"] == 0).all()
    ref = O.solve_lq(synth.random_lq(B, N, n, m, seed=77, kind="dense"))
    for k in ("dx", "du", "dlam"):
        for b in range(B):
            assert rel(g[k][b], ref[k][b]) <= 1e-9, k
