"""Pins of the oracle's LQ adjoint (NEXT-4, oracle_solve_lq_adjoint) against definitions that do not
use it: central finite differences of L(theta) = <g, z(theta)> through the oracle's forward solve
(random directions in every one of the 11 Eq. 4 arrays; symmetric directions for the symmetric
Q, R, P_{N+1}), and the dense KKT solve w = M^-1 g (numpy LAPACK on the assembled Eq. 4 KKT
matrix).  CPU only."""
import numpy as np
import pytest

from tests import kkt_dense
from workloads import synth

KEYS = ("A", "Bm", "c", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0")
SYM = ("Q", "R", "P_term")


def _loss(O, qp, g):
    s = O.solve_lq_single(qp, 0)
    assert s["info"] == 0
    return sum(float((g[k] * s[k]).sum()) for k in ("dx", "du", "dlam")), s


@pytest.mark.parametrize("case", ["dense", "di", "wb"])
def test_adjoint_matches_finite_differences(O, case):
    if case == "dense":
        qp = synth.random_lq(1, 6, 4, 3, seed=3)
    elif case == "di":
        qp = synth.double_integrator(N=8, variant="kkt")
    else:
        qp = synth.random_lq(1, 5, 6, 2, seed=4, kind="wb")
    rng = np.random.default_rng(11)
    N1, n = qp["A"].shape[1:3]
    m = qp["Bm"].shape[-1]
    g = {"dx": rng.standard_normal((N1 + 1, n)), "du": rng.standard_normal((N1, m)),
         "dlam": rng.standard_normal((N1 + 1, n))}
    L0, sol = _loss(O, qp, g)
    grad, info = O.solve_lq_adjoint_single(qp, sol, g)
    assert info == 0
    for k in KEYS:
        E = rng.standard_normal(qp[k][0].shape)
        if k in SYM:
            E = 0.5 * (E + np.swapaxes(E, -1, -2))
        h = 1e-6
        qp_p = {kk: v.copy() for kk, v in qp.items()}; qp_p[k][0] += h * E
        qp_m = {kk: v.copy() for kk, v in qp.items()}; qp_m[k][0] -= h * E
        fd = (_loss(O, qp_p, g)[0] - _loss(O, qp_m, g)[0]) / (2 * h)
        an = float((grad[k] * E).sum())
        assert an == pytest.approx(fd, rel=1e-6, abs=1e-7 * max(1.0, abs(L0))), (k, an, fd)


def test_adjoint_solution_is_dense_kkt_solve(O):
    """w = M^-1 g of the assembled KKT matrix: the vector gradients are -w (q, r, p_{N+1}: primal
    rows; dx0, c: constraint rows)."""
    qp = synth.random_lq(1, 7, 5, 3, seed=8)
    rng = np.random.default_rng(2)
    N = 7; n, m = 5, 3
    g = {"dx": rng.standard_normal((N + 2, n)), "du": rng.standard_normal((N + 1, m)),
         "dlam": rng.standard_normal((N + 2, n))}
    _, sol = _loss(O, qp, g)
    grad, info = O.solve_lq_adjoint_single(qp, sol, g)
    M, _, _ = kkt_dense.assemble(qp, 0)
    gvec = np.concatenate([g["dx"].ravel(), g["du"].ravel(), g["dlam"].ravel()])
    w = np.linalg.solve(M, gvec)
    wx = w[:(N + 2) * n].reshape(N + 2, n)
    wu = w[(N + 2) * n:(N + 2) * n + (N + 1) * m].reshape(N + 1, m)
    wl = w[(N + 2) * n + (N + 1) * m:].reshape(N + 2, n)
    np.testing.assert_allclose(grad["q"], -wx[:N + 1], rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(grad["p_term"], -wx[N + 1], rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(grad["r"], -wu, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(grad["dx0"], -wl[0], rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(grad["c"], -wl[1:], rtol=1e-9, atol=1e-11)
