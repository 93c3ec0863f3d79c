"""Pins of the oracle's SRBD model, barrier, linearisation, cost/theta and line search against
independent definitions: scipy's rotation library, central finite differences, physical special
cases (static equilibrium, free fall, torque-free principal-axis spin, dt=0), the worked barrier
value, and the defining properties of the filter rule.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from workloads import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PRM = synth.srbd_default_params()


def random_state(rng, pitch_max=0.6):
    x = np.zeros(12)
    x[0:3] = rng.uniform(-1, 1, 3); x[2] = 0.3 + 0.05 * rng.standard_normal()
    x[3:6] = [rng.uniform(-0.5, 0.5), rng.uniform(-pitch_max, pitch_max), rng.uniform(-3, 3)]
    x[6:9] = rng.standard_normal(3); x[9:12] = rng.standard_normal(3)
    return x


def random_input(rng):
    u = rng.uniform(-20, 20, 12)
    u[2::3] = rng.uniform(5, 80, 4)
    feet = np.zeros((4, 3)); feet[:, :2] = rng.uniform(-1, 1, (4, 2))
    contact = rng.integers(0, 2, 4).astype(np.uint8)
    return u, feet, contact


def test_rotation_and_euler_kinematics_vs_scipy(O):
    """Theta_dot = E(Theta)^-1 w must make R(Theta(t)) follow Rdot = R [w]_x (body rates), with
    R = Rz(yaw) Ry(pitch) Rx(roll) built by scipy ('ZYX' intrinsic)."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        x = random_state(rng)
        u = np.zeros(12); feet = np.zeros((4, 3)); contact = np.zeros(4, np.uint8)
        xd = O.srbd_f(PRM, x, u, feet, contact)
        eps = 1e-6
        R = lambda th: Rotation.from_euler("ZYX", [th[2], th[1], th[0]]).as_matrix()
        Rdot_fd = (R(x[3:6] + eps * xd[3:6]) - R(x[3:6] - eps * xd[3:6])) / (2 * eps)
        w = x[9:12]
        W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
        assert np.abs(Rdot_fd - R(x[3:6]) @ W).max() < 1e-7


def test_torque_from_single_foot_vs_scipy(O):
    rng = np.random.default_rng(2)
    Iinv = np.linalg.inv(np.array(PRM["inertia"]).reshape(3, 3))
    for _ in range(10):
        x = random_state(rng); x[9:12] = 0
        f = rng.standard_normal(3) * 30
        u = np.zeros(12); u[3:6] = f
        feet = rng.uniform(-1, 1, (4, 3)); contact = np.array([0, 1, 0, 0], np.uint8)
        xd = O.srbd_f(PRM, x, u, feet, contact)
        R = Rotation.from_euler("ZYX", [x[5], x[4], x[3]]).as_matrix()
        tau_w = np.cross(feet[1] - x[0:3], f)
        np.testing.assert_allclose(xd[9:12], Iinv @ (R.T @ tau_w), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(xd[6:9], f / PRM["mass"] + np.array(PRM["gravity"]), atol=1e-13)
        np.testing.assert_allclose(xd[0:3], x[6:9], atol=0)


def test_static_equilibrium(O):
    x = np.zeros(12); x[2] = 0.3
    u = np.zeros(12); u[2::3] = PRM["mass"] * 9.81 / 4
    feet = np.array([[0.19, 0.12, 0], [0.19, -0.12, 0], [-0.19, 0.12, 0], [-0.19, -0.12, 0]], float)
    xd = O.srbd_f(PRM, x, u, feet, np.ones(4, np.uint8))
    assert np.abs(xd[6:12]).max() < 1e-12


def test_free_fall_and_torque_free_spin(O):
    x = np.zeros(12); x[2] = 0.3; x[9:12] = [0.0, 0.0, 2.0]   # spin about a principal axis
    xd = O.srbd_f(PRM, x, np.zeros(12), np.zeros((4, 3)), np.ones(4, np.uint8))
    np.testing.assert_allclose(xd[6:9], PRM["gravity"], atol=1e-15)
    assert np.abs(xd[9:12]).max() < 1e-15
    # swing feet (contact 0) transmit nothing, whatever the force
    u = np.full(12, 50.0)
    xd2 = O.srbd_f(PRM, x, u, np.ones((4, 3)), np.zeros(4, np.uint8))
    np.testing.assert_allclose(xd2, xd, atol=0)


def test_dt_zero_is_identity(O):
    rng = np.random.default_rng(3)
    p = dict(PRM); p["dt"] = 0.0
    x = random_state(rng); u, feet, contact = random_input(rng)
    assert np.array_equal(O.srbd_h(p, x, u, feet, contact), x)


def test_jacobians_vs_central_differences(O):
    rng = np.random.default_rng(4)
    eps = 1e-6
    for _ in range(100):
        x = random_state(rng); u, feet, contact = random_input(rng)
        Fx, Fu = O.srbd_jac(PRM, x, u, feet, contact)
        Fx_fd = np.zeros((12, 12)); Fu_fd = np.zeros((12, 12))
        for k in range(12):
            e = np.zeros(12); e[k] = eps
            Fx_fd[:, k] = (O.srbd_f(PRM, x + e, u, feet, contact) - O.srbd_f(PRM, x - e, u, feet, contact)) / (2 * eps)
            Fu_fd[:, k] = (O.srbd_f(PRM, x, u + e, feet, contact) - O.srbd_f(PRM, x, u - e, feet, contact)) / (2 * eps)
        scale = max(1.0, np.abs(Fx).max())
        assert np.abs(Fx - Fx_fd).max() < 1e-5 * scale
        assert np.abs(Fu - Fu_fd).max() < 1e-5


def test_barrier_worked_value_and_continuity(O):
    g = json.load(open(os.path.join(GOLD, "barrier_value.json")))
    assert O.barrier(g["xi"], g["mu"], g["delta"]) == pytest.approx(g["expected"], abs=g["tol"])
    assert O.barrier(1.0, 1.0, 0.1) == 0.0
    for mu, d in ((1.0, 0.1), (0.1, 1.0), (2.0, 0.5)):
        lo, hi = d * (1 - 1e-12), d * (1 + 1e-12)
        assert O.barrier(lo, mu, d) == pytest.approx(O.barrier(hi, mu, d), abs=1e-9)
        assert O.barrier(d, mu, d) == pytest.approx(-mu * math.log(d), abs=1e-15)
        assert O.barrier_d1(lo, mu, d) == pytest.approx(O.barrier_d1(hi, mu, d), abs=1e-9)
        for xi in np.linspace(d / 10, 10 * d, 57):
            h = 1e-6 * d
            fd1 = (O.barrier(xi + h, mu, d) - O.barrier(xi - h, mu, d)) / (2 * h)
            fd2 = (O.barrier_d1(xi + h, mu, d) - O.barrier_d1(xi - h, mu, d)) / (2 * h)
            assert O.barrier_d1(xi, mu, d) == pytest.approx(fd1, rel=1e-6, abs=1e-6)
            if abs(xi - d) > 2 * h:
                assert O.barrier_d2(xi, mu, d) == pytest.approx(fd2, rel=1e-5, abs=1e-6)


def lagrangian(O, prob, b, x, u, lam):
    """L = J(x,u) + lam_0^T (xhat0 - x_0) + sum_i lam_{i+1}^T (h(x_i,u_i) - x_{i+1})."""
    N = x.shape[0] - 2
    L = O.srbd_cost(prob, b, x, u) + lam[0] @ (prob["x0"][b] - x[0])
    for i in range(N + 1):
        L += lam[i + 1] @ (O.srbd_h(prob["params"], x[i], u[i], prob["feet"][b, i], prob["contact"][b, i]) - x[i + 1])
    return L


def test_linearize_matches_lagrangian_derivatives(O):
    """q = grad_x L, r = grad_u L, p_{N+1} = grad_{x_{N+1}} L, A,B = dh,
    b = h - x_{i+1}, R = d2l/du2 (GN of a linear-in-u barrier is exact), Q = W_x, S = 0."""
    prob = synth.srbd_problem(2, N=6, seed=11)
    rng = np.random.default_rng(5)
    prob["x"] += 0.02 * rng.standard_normal(prob["x"].shape)
    prob["u"] += 3.0 * rng.standard_normal(prob["u"].shape)
    prob["lam"] = rng.standard_normal(prob["lam"].shape)
    lin = O.srbd_linearize(prob, nthreads=1)
    assert (lin["info"] == 0).all()
    eps = 1e-6
    for b in range(2):
        x, u, lam = prob["x"][b].copy(), prob["u"][b].copy(), prob["lam"][b].copy()
        N = 6
        for i in (0, 3, N):
            for k in range(12):
                xp = x.copy(); xm = x.copy(); xp[i, k] += eps; xm[i, k] -= eps
                g = (lagrangian(O, prob, b, xp, u, lam) - lagrangian(O, prob, b, xm, u, lam)) / (2 * eps)
                assert lin["q"][b, i, k] == pytest.approx(g, rel=1e-6, abs=1e-5)
                up = u.copy(); um = u.copy(); up[i, k] += eps; um[i, k] -= eps
                g = (lagrangian(O, prob, b, x, up, lam) - lagrangian(O, prob, b, x, um, lam)) / (2 * eps)
                assert lin["r"][b, i, k] == pytest.approx(g, rel=1e-6, abs=1e-6)
            p = prob["params"]; f_, c_ = prob["feet"][b, i], prob["contact"][b, i]
            hA = np.stack([(O.srbd_h(p, x[i] + e, u[i], f_, c_) - O.srbd_h(p, x[i] - e, u[i], f_, c_)) / (2 * eps)
                           for e in np.eye(12) * eps], axis=1)
            hB = np.stack([(O.srbd_h(p, x[i], u[i] + e, f_, c_) - O.srbd_h(p, x[i], u[i] - e, f_, c_)) / (2 * eps)
                           for e in np.eye(12) * eps], axis=1)
            assert np.abs(lin["A"][b, i] - hA).max() < 1e-7
            assert np.abs(lin["Bm"][b, i] - hB).max() < 1e-9
            np.testing.assert_allclose(lin["c"][b, i], O.srbd_h(p, x[i], u[i], f_, c_) - x[i + 1], atol=1e-14)
            np.testing.assert_allclose(lin["Q"][b, i], np.diag(p["w_x"]), atol=0)
            assert np.abs(lin["S"][b, i]).max() == 0
            # R = Hessian of the stage cost in u (FD of the gradient r at lam = 0)
            prob0 = dict(prob); prob0["lam"] = np.zeros_like(prob["lam"])
            Hu = np.zeros((12, 12))
            for k in range(12):
                up = u.copy(); um = u.copy(); up[i, k] += 1e-4; um[i, k] -= 1e-4
                pp = dict(prob0); pp["u"] = prob["u"].copy(); pp["u"][b] = up
                pm = dict(prob0); pm["u"] = prob["u"].copy(); pm["u"][b] = um
                Hu[:, k] = (O.srbd_linearize(pp, 1)["r"][b, i] - O.srbd_linearize(pm, 1)["r"][b, i]) / 2e-4
            assert np.abs(lin["R"][b, i] - Hu).max() < 1e-6 * max(1.0, np.abs(Hu).max())
        xp = x.copy()
        for k in range(12):
            xp = x.copy(); xm = x.copy(); xp[N + 1, k] += eps; xm[N + 1, k] -= eps
            g = (lagrangian(O, prob, b, xp, u, lam) - lagrangian(O, prob, b, xm, u, lam)) / (2 * eps)
            assert lin["p_term"][b, k] == pytest.approx(g, rel=1e-6, abs=1e-5)
        np.testing.assert_allclose(lin["P_term"][b], np.diag(prob["params"]["w_x_term"]), atol=0)
        np.testing.assert_allclose(lin["dx0"][b], prob["x0"][b] - x[0], atol=0)


def test_linearize_gauss_newton_convexity(O):
    """Every emitted Q, R, P_{N+1} is PSD (SPEC acceptance criterion 6), R SPD."""
    prob = synth.srbd_problem(8, N=20, seed=12)
    prob["u"] += np.random.default_rng(0).normal(0, 30, prob["u"].shape)   # some barriers in the quadratic branch
    lin = O.srbd_linearize(prob)
    assert np.linalg.eigvalsh(lin["Q"]).min() >= -1e-10
    assert np.linalg.eigvalsh(lin["R"]).min() > 0
    assert np.linalg.eigvalsh(lin["P_term"]).min() >= -1e-10


def test_pitch_guard(O):
    prob = synth.srbd_problem(1, N=4, seed=1)
    prob["x"][0, 2, 4] = 1.5
    assert O.srbd_linearize(prob)["info"][0] == -1


def test_theta_definition(O):
    prob = synth.srbd_problem(1, N=5, seed=2)
    p = prob["params"]
    x = prob["x"][0].copy(); u = prob["u"][0]
    # make the trajectory feasible by an exact rollout from xhat0, then add one known defect
    x[0] = prob["x0"][0]
    for i in range(6):
        x[i + 1] = O.srbd_h(p, x[i], u[i], prob["feet"][0, i], prob["contact"][0, i])
    assert O.srbd_theta(prob, 0, x, u) == pytest.approx(0.0, abs=1e-14)
    v = np.array([0.3, 0.0, 0.0, 0, 0, 0, 0, 0, 0, 0, 0, 0])
    x[6] += v
    assert O.srbd_theta(prob, 0, x, u) == pytest.approx(0.3, abs=1e-14)


def accept(J0, th0, g, Ja, tha, alpha, c1, tmax):
    if th0 > tmax:
        return tha <= th0
    if g < 0:
        return Ja <= J0 + c1 * alpha * g
    return Ja < J0 or tha < th0


def test_line_search_selects_largest_accepted(O):
    """Property pin of the filter rule: the returned alpha satisfies the acceptance
    predicate and every larger alpha on the grid violates it."""
    prob = synth.srbd_problem(6, N=12, seed=13)
    rng = np.random.default_rng(7)
    for b in range(6):
        for scale in (0.01, 0.3, 3.0):
            dx = scale * rng.standard_normal((14, 12)) * 0.1
            du = scale * rng.standard_normal((13, 12)) * 10
            j, Ja, tha, (J0, th0, g) = O.srbd_line_search(prob, b, dx, du)
            tmax = 1e-2 * 13
            for jj in range(10):
                ok = accept(J0, th0, g, Ja[jj], tha[jj], 2.0 ** -jj, 1e-4, tmax)
                if j >= 0 and jj < j:
                    assert not ok
                if jj == j:
                    assert ok
            if j < 0:
                assert not any(accept(J0, th0, g, Ja[jj], tha[jj], 2.0 ** -jj, 1e-4, tmax) for jj in range(10))
            # the trial values are the definitions evaluated at x + a dx
            x_a = prob["x"][b] + 0.5 * dx; u_a = prob["u"][b] + 0.5 * du
            assert Ja[1] == pytest.approx(O.srbd_cost(prob, b, x_a, u_a), rel=1e-13)
            assert tha[1] == pytest.approx(O.srbd_theta(prob, b, x_a, u_a), rel=1e-13)


def test_line_search_zero_direction(O):
    prob = synth.srbd_problem(1, N=8, seed=14)
    z_x = np.zeros((10, 12)); z_u = np.zeros((9, 12))
    j, Ja, tha, (J0, th0, g) = O.srbd_line_search(prob, 0, z_x, z_u, theta_max=0.0)   # theta branch
    assert j == 0 and Ja[0] == J0 and tha[0] == th0
    j, *_ = O.srbd_line_search(prob, 0, z_x, z_u, theta_max=1e9)                   # non-descent branch
    assert j == -1


def test_descent_direction_small_alpha_armijo(O):
    """For g < 0 and theta0 <= theta_max, J(a) = J0 + a g + O(a^2) so Armijo with c1 < 1 holds for
    small enough a: the negative cost gradient direction in u must be accepted on the grid."""
    prob = synth.srbd_problem(1, N=8, seed=15)
    b = 0
    u = prob["u"][b]; eps = 1e-6
    gu = np.zeros_like(u)
    for i in range(9):
        for k in range(12):
            up = u.copy(); um = u.copy(); up[i, k] += eps; um[i, k] -= eps
            gu[i, k] = (O.srbd_cost(prob, b, u=up) - O.srbd_cost(prob, b, u=um)) / (2 * eps)
    du = -gu / np.abs(gu).max() * 1.0
    j, Ja, tha, (J0, th0, g) = O.srbd_line_search(prob, b, np.zeros((10, 12)), du, theta_max=1e9)
    assert g < 0 and j >= 0
    assert Ja[j] <= J0 + 1e-4 * 2.0 ** -j * g


def test_step_direction_closes_defects_to_second_order(O):
    """Multiple shooting: the direction satisfies the linearised dynamics, so along
    x + s dx, u + s du the nonlinear defects are (1 - s) * (old defect) + O(s^2): the remainder
    shrinks 4x when s halves."""
    prob = synth.srbd_problem(3, N=20, seed=16)
    p = prob["params"]
    for b in range(3):
        x, u, lam, st, dx, du, dl = O.srbd_step_single(prob, b)
        assert st[4] == 0
        x, u = prob["x"][b], prob["u"][b]
        feet, con = prob["feet"][b], prob["contact"][b]

        def rem(s):
            r = 0.0
            for i in range(21):
                d_new = x[i + 1] + s * dx[i + 1] - O.srbd_h(p, x[i] + s * dx[i], u[i] + s * du[i], feet[i], con[i])
                d_old = x[i + 1] - O.srbd_h(p, x[i], u[i], feet[i], con[i])
                r = max(r, np.abs(d_new - (1 - s) * d_old).max())
            return r
        r1, r2, r3 = rem(0.04), rem(0.02), rem(0.01)
        assert 3.6 < r1 / r2 < 4.4 and 3.6 < r2 / r3 < 4.4


def test_step_batch_matches_single(O):
    prob = synth.srbd_problem(5, N=10, seed=17)
    singles = [O.srbd_step_single(prob, b) for b in range(5)]
    st = O.srbd_step(prob, nthreads=3)
    for b in range(5):
        assert np.array_equal(prob["x"][b], singles[b][0])
        assert np.array_equal(prob["u"][b], singles[b][1])
        assert np.array_equal(prob["lam"][b], singles[b][2])
        assert np.array_equal(st[b], singles[b][3])


def test_solve_zero_iters_is_noop(O):
    """max_iters = 0 returns the iterate unchanged."""
    pr = synth.srbd_problem(2, 20, seed=4)
    x0 = pr["x"].copy()
    it, _ = O.srbd_solve(pr, 0, 1e-8)
    assert (it == 0).all() and np.array_equal(pr["x"], x0)


def test_solve_reaches_fixed_point(O):
    """iterating to convergence reaches a KKT point; one more SQP iteration from
    it moves the trajectory by <= 1e-8 (stationarity) and theta stays <= 1e-10."""
    pr = synth.srbd_problem(3, 30, seed=6)
    it, st = O.srbd_solve(pr, 60, 1e-10)
    assert (it > 0).all() and (it <= 60).all()
    assert (st[:, 1] <= 1e-10).all()
    for b in range(3):
        x, u, lam, s, dx, du, dl = O.srbd_step_single(pr, b)
        assert max(np.abs(x - pr["x"][b]).max(), np.abs(u - pr["u"][b]).max()) <= 1e-8
        assert s[1] <= 1e-10


def test_solve_iteration_count_monotone_in_tol(O):
    """A looser tolerance never needs more iterations (same iterates up to the earlier stop)."""
    a = synth.srbd_problem(4, 30, seed=9)
    b = synth.srbd_problem(4, 30, seed=9)
    ia, _ = O.srbd_solve(a, 60, 1e-4)
    ib, _ = O.srbd_solve(b, 60, 1e-9)
    assert (ia > 0).all() and (ia <= ib).all()


# ----------------------------------------------------------------------------- round-2 pins
def _euler_rates_textbook(Id, w):
    """Euler's rigid-body equations for principal inertias Id = (I1, I2, I3), torque free
    (textbook form, not the cross-product form of the oracle):
    I1 w1' = (I2 - I3) w2 w3,  I2 w2' = (I3 - I1) w3 w1,  I3 w3' = (I1 - I2) w1 w2."""
    I1, I2, I3 = Id
    return np.array([(I2 - I3) * w[1] * w[2] / I1, (I3 - I1) * w[2] * w[0] / I2, (I1 - I2) * w[0] * w[1] / I3])


def test_gyroscopic_term_euler_equations(O):
    """Pins the -w x I w term of P:322-327 (wdot = I^-1(tau - w x I w)) at non-principal spin,
    where it does not vanish: the oracle's wdot must equal Euler's equations written out."""
    rng = np.random.default_rng(41)
    for Id in ((0.10, 0.25, 0.28), (0.3, 0.05, 0.17)):
        p = dict(PRM); p["inertia"] = [Id[0], 0, 0, 0, Id[1], 0, 0, 0, Id[2]]
        for _ in range(10):
            x = random_state(rng)
            xd = O.srbd_f(p, x, np.zeros(12), np.zeros((4, 3)), np.zeros(4, np.uint8))
            np.testing.assert_allclose(xd[9:12], _euler_rates_textbook(Id, x[9:12]), rtol=1e-13, atol=1e-13)
    # one hand-computed value: I = diag(0.1, 0.25, 0.28), w = (1, 2, 3):
    # w1' = (0.25 - 0.28) * 6 / 0.1 = -1.8; w2' = (0.28 - 0.1) * 3 / 0.25 = 2.16; w3' = (0.1 - 0.25) * 2 / 0.28
    x = np.zeros(12); x[2] = 0.3; x[9:12] = [1.0, 2.0, 3.0]
    p = dict(PRM); p["inertia"] = [0.1, 0, 0, 0, 0.25, 0, 0, 0, 0.28]
    xd = O.srbd_f(p, x, np.zeros(12), np.zeros((4, 3)), np.zeros(4, np.uint8))
    np.testing.assert_allclose(xd[9:12], [-1.8, 2.16, -0.3 / 0.28], rtol=1e-14)


def test_torque_free_angular_momentum_conserved(O):
    """Torque-free rigid body (no stance feet), non-principal spin: the world-frame angular
    momentum R(Theta) I w and the kinetic energy 1/2 w^T I w are constants of the motion.  The
    oracle's RK4 plant integrates the oracle's f; a sign error in -w x I w (or in the Euler-angle
    kinematics) breaks conservation by O(1), RK4 at h = 1e-4 s keeps it to ~1e-12."""
    for inertia in ([0.10, 0.0, 0.0, 0.0, 0.25, 0.0, 0.0, 0.0, 0.28],
                    [0.12, 0.01, -0.02, 0.01, 0.20, 0.015, -0.02, 0.015, 0.25]):
        p = dict(PRM); p["inertia"] = inertia
        I = np.array(inertia).reshape(3, 3)
        x = np.zeros(12); x[2] = 0.3; x[3:6] = [0.1, -0.2, 0.3]; x[9:12] = [0.8, -0.6, 1.1]

        def Lw(x):
            R = Rotation.from_euler("ZYX", [x[5], x[4], x[3]]).as_matrix()
            return R @ (I @ x[9:12])
        L0, E0 = Lw(x), 0.5 * x[9:12] @ I @ x[9:12]
        nobody = np.zeros(4, np.uint8)
        for _ in range(50):       # 0.5 s in 50 plant calls of 10 ms, 100 RK4 substeps each
            x = O.srbd_plant(p, x, np.zeros(12), np.zeros((4, 3)), nobody, None, 0.01, 100)
            assert abs(x[4]) < 1.2
            assert np.abs(Lw(x) - L0).max() <= 1e-9 * np.abs(L0).max()
            assert abs(0.5 * x[9:12] @ I @ x[9:12] - E0) <= 1e-9 * E0
        assert np.abs(x[9:12] - [0.8, -0.6, 1.1]).max() > 1e-2     # the body frame rates did change


def test_theta_counts_initial_condition_defect(O):
    """theta = sum_i ||x_{i+1} - h(x_i,u_i)||_2 + ||xhat0 - x_0||_2 (reading R9):
    a ballistic trajectory (no stance feet, w = 0: h(x) = x + dt (v, 0, g, 0), written out here)
    has zero dynamics defects, so theta is exactly the initial-condition term (3-4-5) plus one
    planted defect (5-12-13)."""
    N = 6
    prob = synth.srbd_problem(1, N=N, seed=3)
    p = prob["params"]; dt = p["dt"]; g = np.array(p["gravity"])
    prob["contact"][:] = 0
    x = np.zeros((N + 2, 12)); x[0, 0:3] = [0.1, -0.2, 0.35]; x[0, 3:6] = [0.05, -0.1, 0.7]
    x[0, 6:9] = [0.4, 0.1, 0.0]
    for i in range(N + 1):
        x[i + 1] = x[i]
        x[i + 1, 0:3] = x[i, 0:3] + dt * x[i, 6:9]
        x[i + 1, 6:9] = x[i, 6:9] + dt * g
    u = np.random.default_rng(0).uniform(-5, 5, (N + 1, 12))     # swing feet: forces do nothing
    prob["x0"][0] = x[0]
    assert O.srbd_theta(prob, 0, x, u) == pytest.approx(0.0, abs=1e-14)
    prob["x0"][0] = x[0] + np.r_[0.03, 0.0, 0.0, 0.04, np.zeros(8)]
    assert O.srbd_theta(prob, 0, x, u) == pytest.approx(0.05, abs=1e-14)
    x[N + 1, 6] += 0.05; x[N + 1, 11] += 0.12          # the last node enters one defect only
    assert O.srbd_theta(prob, 0, x, u) == pytest.approx(0.05 + 0.13, abs=1e-14)


def test_cost_value_hand_computed(O):
    """J = sum_i l_i + l_{N+1} on a case computed by hand: tracking terms only
    at the nodes perturbed, one stance foot whose six constraints are written out, the barrier of
    the golden worked value's definition (tests/golden/barrier_value.json)."""
    N = 2
    prob = synth.srbd_problem(1, N=N, seed=4)
    p = prob["params"]
    prob["contact"][:] = 0
    prob["u_ref"][0, 1, 6:9] = 0.0
    x = prob["x_ref"][0].copy(); u = prob["u_ref"][0].copy()
    x[1, 2] += 0.1                         # 1/2 * 500 * 0.01 = 2.5
    x[N + 1, 0] += 0.2                     # terminal: 1/2 * 50 * 0.04 = 1.0
    u[0, 1] += 2.0                         # swing weight 10: 1/2 * 10 * 4 = 20
    prob["contact"][0, 1, 2] = 1           # foot 2 in stance at node 1 with f = (3, -1, 40)
    u[1, 6:9] = [3.0, -1.0, 40.0]          # stance weight 1e-3 against u_ref (0 there: swing)
    track_u = 0.5 * 1e-3 * (9 + 1 + 1600)
    mu, d = p["barrier_mu"], p["barrier_delta"]

    def bar(xi):
        return -mu * math.log(xi) if xi >= d else 0.5 * mu * (((xi - 2 * d) / d) ** 2 - 1) - mu * math.log(d)
    xis = [0.6 * 40 - 3, 0.6 * 40 + 3, 0.6 * 40 + 1, 0.6 * 40 - 1, 40 - 2.0, 250.0 - 40]
    expect = 2.5 + 1.0 + 20.0 + track_u + sum(bar(v) for v in xis)
    assert O.srbd_cost(prob, 0, x, u) == pytest.approx(expect, rel=1e-13)
    # the same foot in the quadratic (relaxed) branch: f_z = 2.5 -> fz - fmin = 0.5 < delta
    u[1, 6:9] = [0.0, 0.0, 2.5]
    xis = [1.5, 1.5, 1.5, 1.5, 0.5, 247.5]
    expect = 2.5 + 1.0 + 20.0 + 0.5 * 1e-3 * 6.25 + sum(bar(v) for v in xis)
    assert O.srbd_cost(prob, 0, x, u) == pytest.approx(expect, rel=1e-13)


def test_cost_slope_matches_central_difference(O):
    """The descent test's slope grad J . (dx, du) (reading R10) equals the central difference of J
    along the direction, with every term active: tracking, terminal, swing weights, and barriers
    in both branches (some stance forces pushed below f_min + delta)."""
    prob = synth.srbd_problem(4, N=10, seed=5)
    rng = np.random.default_rng(9)

    def cd(prob, b, x, u, dx, du):   # central difference, Richardson-extrapolated (O(h^4))
        D = lambda h: (O.srbd_cost(prob, b, x + h * dx, u + h * du) - O.srbd_cost(prob, b, x - h * dx, u - h * du)) / (2 * h)
        return (4 * D(5e-5) - D(1e-4)) / 3
    prob["u"] += rng.normal(0, 8, prob["u"].shape)
    prob["x"] += 0.05 * rng.standard_normal(prob["x"].shape)
    for b in range(4):
        st = prob["contact"][b].astype(bool)
        for i in range(11):
            for j in range(4):
                if st[i, j] and rng.uniform() < 0.3:
                    prob["u"][b, i, 3 * j + 2] = rng.uniform(2.1, 2.9)     # quadratic branch
        for _ in range(3):
            dx = rng.standard_normal((12, 12)) * 0.1
            du = rng.standard_normal((11, 12)) * 2.0
            x, u = prob["x"][b], prob["u"][b]
            fd = cd(prob, b, x, u, dx, du)
            _, _, _, (_, _, g) = O.srbd_line_search(prob, b, dx, du)
            assert g == pytest.approx(fd, rel=1e-7, abs=1e-7 * max(1.0, abs(fd)))
            # terminal-only and u-only directions separately (a dropped term cannot cancel)
            for ddx, ddu in ((np.zeros_like(dx), du), (np.r_[np.zeros((11, 12)), dx[-1:]], np.zeros_like(du))):
                fd = cd(prob, b, x, u, ddx, ddu)
                _, _, _, (_, _, g) = O.srbd_line_search(prob, b, ddx, ddu)
                assert g == pytest.approx(fd, rel=1e-7, abs=1e-7 * max(1.0, abs(fd)))


def test_lm_ladder_recovers_singular_control_weight(O):
    """Levenberg-Marquardt ladder (reading R28): with w_u_swing = 0 the swing-foot block
    of R, hence of G = R + B^T P B (swing columns of B vanish), is singular and the plain iteration
    fails its factorisation (info > 0).  The ladder adds rho = 1e-6 to every R_i, the swing controls
    get a zero step (their gradient is zero) and the solve converges; an accepted step resets rho."""
    prm = dict(synth.srbd_default_params(), w_u_swing=0.0)
    pr = synth.srbd_problem(2, 20, seed=8, params=prm)
    x, u, lam, st, dx, du, dl = O.srbd_step_single(pr, 0)
    assert st[4] > 0 and st[3] == 0
    x, u, lam, st, dx, du, dl = O.srbd_step_single(pr, 0, rho=1e-6)
    assert st[4] == 0 and st[3] == 1
    sw = ~pr["contact"][0].astype(bool)                      # swing feet: zero step
    assert np.abs(du.reshape(21, 4, 3)[sw]).max() < 1e-9
    it, st, rho = O.srbd_solve(pr, 60, 1e-8, return_rho=True)
    assert (it > 0).all() and (st[:, 1] <= 1e-8).all()
    assert (rho <= 1e-6).all()
