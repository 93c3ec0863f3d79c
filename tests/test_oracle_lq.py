"""Pins of the oracle's LQ solve (Riccati Eq. 5 + rollout Eq. 6 + dual Eq. 7) against things
other than itself: the worked scalar example, the dense KKT solve of Eq. 4 (LAPACK), the DARE
closed form (scipy), the discrete Lyapunov special case (scipy), brute-force optimality and
invariants.  CPU only."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

from tests import kkt_dense
from workloads import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-30)


def scalar_problem(dx0=1.0):
    one = lambda *s: np.ones((1,) + s)
    return {"A": one(1, 1, 1), "Bm": one(1, 1, 1), "c": np.zeros((1, 1, 1)), "Q": one(1, 1, 1),
            "R": one(1, 1, 1), "S": np.zeros((1, 1, 1, 1)), "q": np.zeros((1, 1, 1)), "r": np.zeros((1, 1, 1)),
            "P_term": one(1, 1), "p_term": np.zeros((1, 1)), "dx0": np.full((1, 1), dx0)}


def test_scalar_worked_example(O):
    g = json.load(open(os.path.join(GOLD, "scalar_one_step.json")))["expected"]
    out = O.solve_lq_single(scalar_problem())
    assert out["info"] == 0
    assert out["K"][0, 0, 0] == pytest.approx(g["K0"], abs=1e-15)
    assert out["k"][0, 0] == pytest.approx(g["k0"], abs=1e-15)
    assert out["P"][0, 0, 0] == pytest.approx(g["P0"], abs=1e-15)
    assert out["P"][1, 0, 0] == pytest.approx(g["P1"], abs=1e-15)
    assert out["p"][0, 0] == pytest.approx(g["p0"], abs=1e-15)
    np.testing.assert_allclose(out["du"].ravel(), g["du"], atol=1e-15)
    np.testing.assert_allclose(out["dx"].ravel(), g["dx"], atol=1e-15)
    np.testing.assert_allclose(out["dlam"].ravel(), g["dlam"], atol=1e-15)


def test_scalar_example_matches_dense_kkt():
    g = json.load(open(os.path.join(GOLD, "scalar_one_step.json")))["expected"]
    dx, du, lam = kkt_dense.solve(scalar_problem())
    np.testing.assert_allclose(dx.ravel(), g["dx"], atol=1e-14)
    np.testing.assert_allclose(du.ravel(), g["du"], atol=1e-14)
    np.testing.assert_allclose(lam.ravel(), g["dlam"], atol=1e-14)


@pytest.mark.parametrize("case", [
    ("di", 32, 4, 2), ("dense", 0, 3, 2), ("dense", 1, 3, 2), ("dense", 8, 4, 3),
    ("dense", 16, 5, 1), ("dense", 12, 12, 12), ("wb", 10, 8, 4),
])
def test_riccati_matches_dense_kkt(O, case):
    kind, N, n, m = case
    qp = synth.double_integrator(N, variant="kkt") if kind == "di" else synth.random_lq(2, N, n, m, kind=kind)
    for b in range(qp["A"].shape[0]):
        out = O.solve_lq_single(qp, b)
        assert out["info"] == 0
        dx, du, lam = kkt_dense.solve(qp, b)
        assert rel(out["dx"], dx) < 1e-9
        assert rel(out["du"], du) < 1e-9
        assert rel(out["dlam"], lam) < 1e-9
        assert kkt_dense.backward_error(qp, b, out["dx"], out["du"], out["dlam"]) < 1e-14
        assert kkt_dense.backward_error_blockwise(qp, b, out["dx"], out["du"], out["dlam"]) < 1e-14


def di_dare():
    qp = synth.double_integrator(32, variant="dare")
    A, Bm, Q, R = qp["A"][0, 0], qp["Bm"][0, 0], qp["Q"][0, 0], qp["R"][0, 0]
    Pinf = sla.solve_discrete_are(A, Bm, Q, R)
    qp["P_term"] = Pinf[None].copy()
    Kinf = -np.linalg.solve(R + Bm.T @ Pinf @ Bm, Bm.T @ Pinf @ A)
    return qp, Pinf, Kinf


def test_dare_fixed_point(O):
    qp, Pinf, Kinf = di_dare()
    out = O.solve_lq_single(qp)
    for i in range(33 + 1):
        assert rel(out["P"][i], Pinf) < 1e-12
    for i in range(33):
        assert rel(out["K"][i], Kinf) < 1e-12
    A, Bm = qp["A"][0, 0], qp["Bm"][0, 0]
    Acl = A + Bm @ Kinf
    x = qp["dx0"][0].copy()
    for i in range(34):
        assert np.abs(out["dx"][i] - x).max() < 1e-12
        x = Acl @ x


def test_dare_optimal_cost_golden(O):
    g = json.load(open(os.path.join(GOLD, "dare_cost.json")))
    qp, Pinf, _ = di_dare()
    out = O.solve_lq_single(qp)
    # cost of the oracle's trajectory, evaluated from the Eq. 4 objective directly
    Q, R = qp["Q"][0, 0], qp["R"][0, 0]
    f = sum(0.5 * out["dx"][i] @ Q @ out["dx"][i] + 0.5 * out["du"][i] @ R @ out["du"][i] for i in range(33))
    f += 0.5 * out["dx"][33] @ Pinf @ out["dx"][33]
    x0 = np.array(g["dx0"])
    assert f == pytest.approx(0.5 * x0 @ Pinf @ x0, rel=1e-12)
    assert f == pytest.approx(g["expected_cost"], abs=g["tol"])


def test_lyapunov_special_case(O):
    """B = 0 (no control authority): P_i = Q + A^T P_{i+1} A; with P_{N+1} the solution of the
    discrete Lyapunov equation P = A^T P A + Q (scipy) every P_i is that solution."""
    rng = np.random.default_rng(3)
    n, m, N = 5, 2, 20
    A0 = rng.standard_normal((n, n)); A0 *= 0.9 / np.max(np.abs(np.linalg.eigvals(A0)))
    Q0 = np.diag(rng.uniform(0.5, 2.0, n))
    Pl = sla.solve_discrete_lyapunov(A0.T, Q0)
    qp = synth.random_lq(1, N, n, m)
    qp["A"][:] = A0; qp["Bm"][:] = 0; qp["Q"][:] = Q0; qp["S"][:] = 0; qp["P_term"][0] = Pl
    qp["q"][:] = 0; qp["r"][:] = 0; qp["c"][:] = 0; qp["p_term"][:] = 0
    out = O.solve_lq_single(qp)
    for i in range(N + 2):
        assert rel(out["P"][i], Pl) < 1e-11
    assert np.abs(out["K"]).max() == 0.0


def test_zero_cost_fixed_point(O):
    qp = synth.random_lq(1, 6, 4, 3)
    for k in ("Q", "S", "q", "r", "P_term", "p_term"):
        qp[k][:] = 0
    qp["R"][:] = np.eye(3)
    out = O.solve_lq_single(qp)
    for k in ("K", "k", "P", "p"):
        assert np.abs(out[k]).max() == 0.0


def test_brute_force_optimality(O):
    """The oracle's (dx, du) is feasible and no random feasible perturbation has lower cost."""
    qp = synth.random_lq(1, 6, 3, 2)
    out = O.solve_lq_single(qp)
    A, Bm, c = qp["A"][0], qp["Bm"][0], qp["c"][0]

    def cost(du):
        x = qp["dx0"][0].copy(); f = 0.0
        for i in range(7):
            z = np.concatenate([x, du[i]])
            H = np.block([[qp["Q"][0, i], qp["S"][0, i].T], [qp["S"][0, i], qp["R"][0, i]]])
            f += 0.5 * z @ H @ z + qp["q"][0, i] @ x + qp["r"][0, i] @ du[i]
            x = A[i] @ x + Bm[i] @ du[i] + c[i]
        return f + 0.5 * x @ qp["P_term"][0] @ x + qp["p_term"][0] @ x

    f0 = cost(out["du"])
    rng = np.random.default_rng(0)
    for _ in range(200):
        assert cost(out["du"] + 1e-3 * rng.standard_normal(out["du"].shape)) > f0


def test_kkt_invariants_long_horizon(O):
    qp = synth.random_lq(1, 400, 12, 12)
    out = O.solve_lq_single(qp)
    assert kkt_dense.backward_error_blockwise(qp, 0, out["dx"], out["du"], out["dlam"]) < 1e-13
    for i in range(402):
        assert np.abs(out["P"][i] - out["P"][i].T).max() <= 1e-9 * np.abs(out["P"][i]).max()


def test_failure_names_stage(O):
    qp = synth.random_lq(1, 5, 3, 2)
    qp["R"][0, 3] = -10 * np.eye(2)     # G_3 = R_3 + B^T P B indefinite
    out = O.solve_lq_single(qp)
    assert out["info"] == 1 + 3


def test_batch_equals_single(O):
    qp = synth.random_lq(5, 7, 4, 3)
    bat = O.solve_lq(qp, nthreads=2)
    for b in range(5):
        s = O.solve_lq_single(qp, b)
        assert np.array_equal(bat["dx"][b], s["dx"]) and np.array_equal(bat["dlam"][b], s["dlam"])
    assert (bat["info"] == 0).all()
