"""Pins of the oracle's centralized multi-robot model (NEXT-3, oracle_multi_*) against definitions
that do not use it: separability without coupling (block-diagonal KKT: the joint direction equals
the per-robot directions of the single-robot oracle), the collision cost's gradient and
Gauss-Newton Hessian against central finite differences of the cost (single pair: GN Hessian =
grad J grad J^T / (2 J) exactly), the linearisation against finite differences of the joint
Lagrangian, the cost slope against finite differences, and theta on a ballistic trajectory.
CPU only."""
import math

import numpy as np
import pytest

from workloads import synth


def problem(B=2, R=4, N=6, seed=3, w=None, spacing=1.2):
    p = synth.multi_srbd_problem(B, R, N=N, seed=seed, spacing=spacing)
    if w is not None:
        p["multi"] = dict(p["multi"], weight=w)
    return p


def robot(p, b, k):
    """Single-robot problem dict of robot k of instance b (indexing only)."""
    R = p["multi"]["n_robots"]
    sl = slice(12 * k, 12 * k + 12)
    q = {"params": p["params"]}
    for key in ("x", "u", "lam", "x_ref", "u_ref"):
        q[key] = np.ascontiguousarray(p[key][b:b + 1, :, sl])
    q["x0"] = np.ascontiguousarray(p["x0"][b:b + 1, sl])
    q["contact"] = np.ascontiguousarray(p["contact"][b:b + 1, :, 4 * k:4 * k + 4])
    q["feet"] = np.ascontiguousarray(p["feet"][b:b + 1, :, 4 * k:4 * k + 4])
    assert R > k
    return q


def test_separable_without_coupling(O):
    p = problem(w=0.0)
    for b in range(2):
        _, _, _, st, dx, du, dl = O.multi_step_single(p, b)
        assert st[4] == 0
        lin = O.multi_linearize_single(p, b)
        for k in range(4):
            q = robot(p, b, k)
            _, _, _, st1, dx1, du1, dl1 = O.srbd_step_single(q, 0)
            sl = slice(12 * k, 12 * k + 12)
            np.testing.assert_allclose(dx[:, sl], dx1, rtol=1e-9, atol=1e-12)
            np.testing.assert_allclose(du[:, sl], du1, rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(dl[:, sl], dl1, rtol=1e-9, atol=1e-9)
            l1 = O.srbd_linearize(q, nthreads=1)
            np.testing.assert_allclose(lin["Q"][:, sl, sl], l1["Q"][0], atol=0)
            np.testing.assert_allclose(lin["A"][:, sl, sl], l1["A"][0], atol=0)
        # off-diagonal blocks vanish
        mask = np.kron(np.eye(4), np.ones((12, 12))) == 0
        for key in ("A", "Bm", "Q", "R"):
            assert np.abs(lin[key][:, mask]).max() == 0


def test_collision_gradient_and_gauss_newton_single_pair(O):
    """R = 2 robots close together: q_coll = grad J_coll (central differences of the oracle's
    collision cost), Q_coll = w grad eps grad eps^T = grad J grad J^T / (2 J) (J = w eps^2 / 2)."""
    p = problem(B=1, R=2, N=3, seed=5, spacing=0.7)
    lin = O.multi_linearize_single(p, 0)
    p0 = dict(p, multi=dict(p["multi"], weight=0.0))
    lin0 = O.multi_linearize_single(p0, 0)
    for i in range(5):      # stages 0..3 (Q_i, q_i) and the terminal node 4 (P_{N+1}, p_{N+1})
        x = p["x"][0, i].copy()
        J = O.multi_coll_cost(p["multi"], x)
        assert J > 1e-3
        g = np.zeros(24)
        for k in range(24):
            e = np.zeros(24); e[k] = 1e-6
            g[k] = (O.multi_coll_cost(p["multi"], x + e) - O.multi_coll_cost(p["multi"], x - e)) / 2e-6
        if i <= 3:
            qc = lin["q"][i] - lin0["q"][i]
            Qc = lin["Q"][i] - lin0["Q"][i]
        else:
            qc = lin["p_term"] - lin0["p_term"]
            Qc = lin["P_term"] - lin0["P_term"]
        np.testing.assert_allclose(qc, g, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(Qc, np.outer(g, g) / (2 * J), rtol=1e-6, atol=1e-6)
        assert set(np.nonzero(np.abs(g) > 0)[0]) <= {0, 1, 12, 13}


def lagrangian(O, p, b, x, u, lam):
    """L = J(x,u) + lam_0^T (xhat0 - x_0) + sum_i lam_{i+1}^T (h(x_i,u_i) - x_{i+1}), h per robot."""
    N = x.shape[0] - 2
    R = p["multi"]["n_robots"]
    L = O.multi_cost(p, b, x, u) + lam[0] @ (p["x0"][b] - x[0])
    for i in range(N + 1):
        for k in range(R):
            sl = slice(12 * k, 12 * k + 12)
            hk = O.srbd_h(p["params"], x[i, sl], u[i, sl], p["feet"][b, i, 4 * k:4 * k + 4], p["contact"][b, i, 4 * k:4 * k + 4])
            L += lam[i + 1, sl] @ (hk - x[i + 1, sl])
    return L


def test_linearize_matches_joint_lagrangian(O):
    p = problem(B=1, R=3, N=4, seed=7, spacing=1.0)
    rng = np.random.default_rng(2)
    p["lam"] = rng.standard_normal(p["lam"].shape)
    p["u"] += rng.standard_normal(p["u"].shape)
    lin = O.multi_linearize_single(p, 0)
    x, u, lam = p["x"][0].copy(), p["u"][0].copy(), p["lam"][0].copy()
    eps = 1e-6
    for i in (0, 2, 4):
        for k in (0, 1, 5, 12, 13, 25, 30):
            xp = x.copy(); xm = x.copy(); xp[i, k] += eps; xm[i, k] -= eps
            g = (lagrangian(O, p, 0, xp, u, lam) - lagrangian(O, p, 0, xm, u, lam)) / (2 * eps)
            assert lin["q"][i, k] == pytest.approx(g, rel=1e-6, abs=1e-5)
            up = u.copy(); um = u.copy(); up[i, k] += eps; um[i, k] -= eps
            g = (lagrangian(O, p, 0, x, up, lam) - lagrangian(O, p, 0, x, um, lam)) / (2 * eps)
            assert lin["r"][i, k] == pytest.approx(g, rel=1e-6, abs=1e-6)
    for k in (0, 13, 35):
        xp = x.copy(); xm = x.copy(); xp[5, k] += eps; xm[5, k] -= eps
        g = (lagrangian(O, p, 0, xp, u, lam) - lagrangian(O, p, 0, xm, u, lam)) / (2 * eps)
        assert lin["p_term"][k] == pytest.approx(g, rel=1e-6, abs=1e-5)


def test_cost_slope_matches_finite_difference(O):
    p = problem(B=1, R=3, N=5, seed=9, spacing=0.9)
    rng = np.random.default_rng(4)
    for _ in range(3):
        dx = 0.05 * rng.standard_normal(p["x"][0].shape)
        du = 2.0 * rng.standard_normal(p["u"][0].shape)
        x, u = p["x"][0], p["u"][0]
        D = lambda h: (O.multi_cost(p, 0, x + h * dx, u + h * du) - O.multi_cost(p, 0, x - h * dx, u - h * du)) / (2 * h)
        fd = (4 * D(5e-5) - D(1e-4)) / 3
        assert O.multi_cost_slope(p, 0, dx, du) == pytest.approx(fd, rel=1e-7, abs=1e-7 * max(1.0, abs(fd)))


def test_theta_ballistic_plus_planted_defect(O):
    """No stance feet, w = 0: h(x) = x + dt (v, 0, g, 0) per robot (written out here); theta is the
    stacked initial-condition defect (3-4-5) plus one planted stacked defect (5-12-13) across two robots."""
    p = problem(B=1, R=2, N=4, seed=1)
    p["contact"][:] = 0
    dt = p["params"]["dt"]; g = np.array(p["params"]["gravity"])
    x = np.zeros((6, 24))
    x[0, 0:3] = [0.1, 0.2, 0.3]; x[0, 6:9] = [0.3, -0.1, 0.0]
    x[0, 12:15] = [1.1, 0.2, 0.3]; x[0, 18:21] = [-0.2, 0.4, 0.1]
    for i in range(5):
        x[i + 1] = x[i]
        for o in (0, 12):
            x[i + 1, o:o + 3] = x[i, o:o + 3] + dt * x[i, o + 6:o + 9]
            x[i + 1, o + 6:o + 9] = x[i, o + 6:o + 9] + dt * g
    u = np.random.default_rng(0).uniform(-5, 5, (5, 24))
    p["x0"][0] = x[0]
    assert O.multi_theta(p, 0, x, u) == pytest.approx(0.0, abs=1e-14)
    p["x0"][0] = x[0] + np.r_[0.03, np.zeros(12), 0.04, np.zeros(10)]
    assert O.multi_theta(p, 0, x, u) == pytest.approx(0.05, abs=1e-14)
    x[5, 6] += 0.05; x[5, 23] += 0.12
    assert O.multi_theta(p, 0, x, u) == pytest.approx(0.05 + 0.13, abs=1e-14)
