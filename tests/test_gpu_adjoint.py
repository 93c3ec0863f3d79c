"""GPU parity of the LQ adjoint (NEXT-4, pdilqr_solve_lq_adjoint) against the fp64 oracle's adjoint
(itself pinned by finite differences and the dense KKT solve, tests/test_oracle_adjoint.py) on
identical seeded, dtype-rounded inputs, and the torch.autograd wrapper end to end."""
import numpy as np
import pytest
import torch

from tests.gpu_util import rel, rounded, to_np
from workloads import synth

pytestmark = pytest.mark.gpu
KEYS = ("A", "Bm", "c", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def _dev(d, dtype):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", dtype) for k, v in d.items()
            if isinstance(v, np.ndarray)}


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("case,B,N,n,m,chunk", [("dense", 5, 20, 12, 12, 0), ("dense", 3, 9, 5, 3, 1),
                                                ("dense", 200, 30, 8, 4, 0), ("wb", 2, 12, 74, 32, 0),
                                                ("dense", 2, 0, 4, 2, 0), ("dense", 2, 1, 3, 3, 1),
                                                ("dense", 2, 7, 40, 24, 0)])
def test_adjoint_parity(P, O, dtype, case, B, N, n, m, chunk):
    qp = rounded(synth.random_lq(B, N, n, m, seed=17 + n, kind=case), dtype)
    rng = np.random.default_rng(5)
    g = rounded({"dx": rng.standard_normal((B, N + 2, n)), "du": rng.standard_normal((B, N + 1, m)),
                 "dlam": rng.standard_normal((B, N + 2, n))}, dtype)
    h = P.PdIlqr(N=N, n=n, m=m, batch=B, dtype=dtype, leaf_chunk=chunk)
    dq = _dev(qp, dtype)
    sol = h.solve_lq(dq)
    grad = h.solve_lq_adjoint(dq, sol, _dev(g, dtype))
    torch.cuda.synchronize()
    assert (to_np(grad["info"]) == 0).all()
    tol = 1e-4 if dtype == torch.float32 else 1e-9
    for b in range(min(B, 6)):
        s_ref = O.solve_lq_single(qp, b)
        ref, info = O.solve_lq_adjoint_single(qp, s_ref, {k: g[k][b] for k in g}, b)
        assert info == 0
        for k in KEYS:
            e = rel(to_np(grad[k][b]), ref[k])
            assert e <= tol, (k, b, e)


def test_autograd_end_to_end(P, O):
    """loss = sum(w_x * dx) + sum(w_u * du): torch.autograd through lq_solve gives the oracle's
    adjoint gradients for every Eq. 4 input (fp64)."""
    B, N, n, m = 2, 10, 6, 3
    qp = synth.random_lq(B, N, n, m, seed=23)
    dq = {k: v.requires_grad_(True) for k, v in _dev(qp, torch.float64).items()}
    h = P.PdIlqr(N=N, n=n, m=m, batch=B, dtype=torch.float64)
    dx, du, dlam, info = P.lq_solve(h, dq)
    rng = np.random.default_rng(3)
    wx = torch.from_numpy(rng.standard_normal(dx.shape)).cuda()
    wu = torch.from_numpy(rng.standard_normal(du.shape)).cuda()
    loss = (wx * dx).sum() + (wu * du).sum()
    loss.backward()
    assert (info == 0).all()
    for b in range(B):
        s_ref = O.solve_lq_single(qp, b)
        ref, _ = O.solve_lq_adjoint_single(qp, s_ref, {"dx": wx[b].cpu().numpy(), "du": wu[b].cpu().numpy(),
                                                       "dlam": None}, b)
        for k in KEYS:
            assert rel(to_np(dq[k].grad[b]), ref[k]) <= 1e-9, k
