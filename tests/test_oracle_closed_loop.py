"""Pins for the oracle's closed-loop pieces: warm-start shift (P:315,
SPEC S:343-350), RK4 SRBD plant with an external force and the closed-loop
RTI scenarios of SPEC S:518-521 (measured on the oracle, fp64)."""
import numpy as np
import pytest

from workloads import synth


def test_shift_definition(O):
    a = np.arange(3.0)[:, None] * np.ones((1, 12))          # x = (a, b, c)
    s = O.warm_start_shift(a)
    assert np.array_equal(s[0], a[1]) and np.array_equal(s[1], a[2]) and np.array_equal(s[2], a[2])
    c = np.ones((4, 5, 12)) * 7.0                             # constant trajectory: unchanged
    assert np.array_equal(O.warm_start_shift(c), c)


def _no_contact():
    return np.zeros(12), np.zeros(12), np.zeros(4, np.uint8)


@pytest.mark.parametrize("sub", [1, 3])
def test_plant_free_flight_closed_form(O, sub):
    """No contact, external force F: p(t) = p0 + v0 t + (g + F/m) t^2 / 2 exactly (RK4 is exact on
    polynomials of degree <= 4); the attitude with w = 0 stays put."""
    prm = synth.srbd_default_params()
    rng = np.random.default_rng(3)
    x = rng.normal(size=12) * 0.3
    x[9:] = 0.0
    u, feet, con = _no_contact()
    F = np.array([15.0, -7.0, 30.0])
    t = 0.1
    y = O.srbd_plant(prm, x, u, feet, con, F, t, sub)
    acc = np.array(prm["gravity"]) + F / prm["mass"]
    np.testing.assert_allclose(y[0:3], x[0:3] + x[6:9] * t + 0.5 * acc * t * t, rtol=0, atol=1e-14)
    np.testing.assert_allclose(y[6:9], x[6:9] + acc * t, rtol=0, atol=1e-14)
    np.testing.assert_allclose(y[3:6], x[3:6], rtol=0, atol=0)


def test_plant_principal_axis_spin(O):
    """Torque-free spin about the body z principal axis, level attitude: w constant (w x Iw = 0),
    yaw(t) = yaw0 + w t exactly."""
    prm = synth.srbd_default_params()
    x = np.zeros(12); x[5] = 0.4; x[11] = 1.7
    u, feet, con = _no_contact()
    y = O.srbd_plant(prm, x, u, feet, con, None, 0.3, 2)
    assert abs(y[5] - (0.4 + 1.7 * 0.3)) < 1e-14 and abs(y[11] - 1.7) < 1e-15
    assert np.abs(y[3:5]).max() == 0.0


def test_plant_static_equilibrium(O):
    """Four feet symmetric about the CoM, each pushing m g / 4 straight up: f(x, u) = 0."""
    prm = synth.srbd_default_params()
    x = np.zeros(12); x[0:3] = (0.2, -0.1, 0.3)
    feet = np.array([[0.2 + sx * 0.2, -0.1 + sy * 0.15, 0.0] for sx, sy in ((1, 1), (1, -1), (-1, 1), (-1, -1))]).ravel()
    u = np.zeros(12); u[2::3] = prm["mass"] * -prm["gravity"][2] / 4
    y = O.srbd_plant(prm, x, u, feet, np.ones(4, np.uint8), None, 0.5, 5)
    np.testing.assert_allclose(y, x, rtol=0, atol=1e-13)


def test_plant_fourth_order(O):
    """RK4 global error O(h^4): halving h cuts the error ~16x (vs a fine-step solution)."""
    prm = synth.srbd_default_params()
    pr = synth.srbd_problem(1, 10, seed=11)
    x, u, feet, con = pr["x0"][0], pr["u"][0, 0] * 1.3, pr["feet"][0, 0].ravel(), pr["contact"][0, 0]
    x = x.copy(); x[9:] = (0.8, -0.6, 1.1)
    fine = O.srbd_plant(prm, x, u, feet, con, None, 0.1, 4096)
    e1 = np.abs(O.srbd_plant(prm, x, u, feet, con, None, 0.1, 4) - fine).max()
    e2 = np.abs(O.srbd_plant(prm, x, u, feet, con, None, 0.1, 8) - fine).max()
    assert 14.0 < e1 / e2 < 18.0, (e1, e2)


def test_plant_euler_consistency(O):
    """One tiny RK4 step agrees with x + h f(x) to O(h^2) (plant and oracle_srbd_f are one model)."""
    prm = synth.srbd_default_params()
    pr = synth.srbd_problem(1, 10, seed=12)
    x, u, feet, con = pr["x0"][0], pr["u"][0, 0], pr["feet"][0, 0].ravel(), pr["contact"][0, 0]
    h = 1e-6
    y = O.srbd_plant(prm, x, u, feet, con, None, h, 1)
    f = O.srbd_f(prm, x, u, feet, con)
    np.testing.assert_allclose((y - x) / h, f, rtol=0, atol=1e-3 * np.abs(f).max())


T4 = 200   # 4 s at 50 Hz


def test_closed_loop_trot_tracking(O):
    """0.3 m/s trot, no disturbance, 4 s -> mean forward-velocity error < 0.1 m/s."""
    L = synth.srbd_problem(1, 50 + T4, seed=1, randomize=False, v_cmd=(0.3, 0.0))
    r = O.closed_loop(L, 50, T4)
    assert np.abs(r["x_plant"][0, :, 6] - 0.3).mean() < 0.1
    assert (r["stats"][0, :, 4] == 0).all() and (r["stats"][0, :, 3] == 1).all()


def test_closed_loop_station_keeping(O):
    """zero command, 4 s -> base position drift < 0.05 m."""
    L = synth.srbd_problem(1, 50 + T4, seed=1, randomize=False, v_cmd=(0.0, 0.0))
    r = O.closed_loop(L, 50, T4)
    assert np.linalg.norm(r["x_plant"][0, -1, :2] - r["x_plant"][0, 0, :2]) < 0.05


def test_closed_loop_push_recovery(O):
    """SPEC S:519 / P:388 lateral push, at the impulse the fixed-foothold controller absorbs
    (reading R23: 50 N for 0.12 s; footholds are open-loop inputs, no Raibert feedback):
    vy returns within 0.1 m/s of the command within 1.0 s after the push ends."""
    T = 150
    L = synth.srbd_problem(1, 50 + T, seed=1, randomize=False, v_cmd=(0.3, 0.0))
    push = lambda node: np.array([[0.0, 50.0, 0.0]]) if 50 <= node < 56 else None
    r = O.closed_loop(L, 50, T, push=push)
    vy = r["x_plant"][0, :, 7]
    assert vy[53:58].max() > 0.2                       # the push did act
    assert np.abs(vy[56 + 50:]).max() < 0.1


def test_closed_loop_25hz(O):
    """nodes_per_tick = 2 (25 Hz control on 20 ms nodes) stays stable and tracks."""
    T = 100
    L = synth.srbd_problem(1, 50 + 2 * T, seed=1, randomize=False, v_cmd=(0.3, 0.0))
    r = O.closed_loop(L, 50, T, nodes_per_tick=2)
    assert np.isfinite(r["x_plant"]).all()
    assert r["x_plant"].shape[1] == 2 * T + 1
    assert np.abs(r["x_plant"][0, :, 6] - 0.3).mean() < 0.1
    assert abs(r["x_plant"][0, -1, 0] - L["x_ref"][0, 2 * T, 0]) < 0.05
