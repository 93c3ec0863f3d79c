"""GPU parity of the closed-loop RTI pieces: pdilqr_shift (bit-exact),
pdilqr_srbd_plant (RK4 + external force) and whole closed loops (ClosedLoop: step + plant + shift
per node) against the oracle's closed_loop (oracle/oracle.py), fp64 and fp32."""
import numpy as np
import pytest
import torch

from tests.gpu_util import to_np
from workloads import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def dev(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype == torch.float64:
        t = t.to(dtype)
    return t.cuda().contiguous()


def handle(P, B, N, dtype, prm):
    return P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=dtype, model="srbd", srbd=prm)


def iterate(pr, N, dtype):
    it = {k: dev(pr[k][:, :N + 2], dtype) for k in ("x", "lam", "x_ref")}
    it.update({k: dev(pr[k][:, :N + 1], dtype) for k in ("u", "u_ref", "contact", "feet")})
    it["x0"] = dev(pr["x0"], dtype)
    return it


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_shift_bitexact(P, O, dtype):
    B, N = 37, 23
    pr = synth.srbd_problem(B, N, seed=4)
    rng = np.random.default_rng(0)
    for k in ("x", "u", "lam"):
        pr[k] = pr[k] + rng.normal(size=pr[k].shape)
    h = handle(P, B, N, dtype, pr["params"])
    it = iterate(pr, N, dtype)
    ref = {k: O.warm_start_shift(to_np(it[k])) for k in ("x", "u", "lam")}
    h.shift(it)
    torch.cuda.synchronize()
    for k in ref:
        assert np.array_equal(to_np(it[k]), ref[k]), k


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 2e-5)])
def test_plant_parity(P, O, dtype, tol):
    B, N = 300, 5
    pr = synth.srbd_problem(B, N, seed=8)
    rng = np.random.default_rng(1)
    xp = pr["x0"] + 0.1 * rng.normal(size=(B, 12))
    uh = pr["u"][:, 0] * (1 + 0.3 * rng.normal(size=(B, 12)))
    F = 40 * rng.normal(size=(B, 3))
    F[::3] = 0
    h = handle(P, B, N, dtype, pr["params"])
    it = iterate(pr, N, dtype)
    x_d, u_d, F_d = dev(xp, dtype), dev(uh, dtype), dev(F, dtype)
    # both sides consume the dtype-rounded inputs
    xq, uq, Fq = to_np(x_d), to_np(u_d), to_np(F_d)
    fq = to_np(it["feet"])[:, 0].reshape(B, 12)
    h.plant(it, x_d, u_d, F_d, dt=0.02, substeps=4)
    torch.cuda.synchronize()
    got = to_np(x_d)
    for b in range(B):
        ref = O.srbd_plant(pr["params"], xq[b], uq[b], fq[b], pr["contact"][b, 0], Fq[b], 0.02, 4)
        err = np.abs(got[b] - ref).max() / max(1.0, np.abs(ref).max())
        assert err <= tol, (b, err)
    # NULL external force == zero force
    x2 = dev(xp, dtype)
    h.plant(it, x2, u_d, None, dt=0.02, substeps=4)
    x3 = dev(xp, dtype)
    h.plant(it, x3, u_d, torch.zeros_like(F_d), dt=0.02, substeps=4)
    torch.cuda.synchronize()
    assert torch.equal(x2, x3)


def run_gpu_loop(P, L, N, ticks, dtype, k=1, push=None):
    B = L["x0"].shape[0]
    h = handle(P, B, N, dtype, L["params"])
    ref = {"x_ref": dev(L["x_ref"], dtype), "u_ref": dev(L["u_ref"], dtype),
           "contact": dev(L["contact"], dtype), "feet": dev(L["feet"], dtype)}
    it0 = {"x": dev(L["x"][:, :N + 2], dtype), "u": dev(L["u"][:, :N + 1], dtype), "lam": dev(L["lam"][:, :N + 2], dtype)}
    cl = P.ClosedLoop(h, ref, it0, dev(L["x0"], dtype), nodes_per_tick=k)
    xs, sts = [to_np(cl.x_plant)], []
    pushf = None if push is None else (lambda node: None if push(node) is None else dev(push(node), dtype))
    for _ in range(ticks):
        st = cl.tick(pushf)
        sts.append(np.stack([to_np(st[c]).astype(np.float64) for c in ("cost", "theta", "alpha", "accepted", "info")], 1))
        xs.append(to_np(cl.x_plant))
    return np.stack(xs, 1), np.stack(sts, 1)


@pytest.mark.parametrize("k", [1, 2])
def test_closed_loop_fp64_matches_oracle(P, O, k):
    """fp64: the GPU closed loop follows the oracle's closed loop node by node (same alphas)."""
    N, T = 30, 25
    L = synth.round_to(synth.srbd_problem(4, N + k * T + 1, seed=21), np.float64)
    r = O.closed_loop(L, N, T, nodes_per_tick=k)
    xs, sts = run_gpu_loop(P, L, N, T, torch.float64, k)
    xo = r["x_plant"][:, ::k]
    assert np.abs(xs - xo).max() <= 1e-8 * max(1.0, np.abs(xo).max())
    assert np.array_equal(sts[..., 2], r["stats"][..., 2])          # same line-search decisions
    assert (sts[..., 4] == 0).all()


def test_closed_loop_fp32_tracks_oracle(P, O):
    """fp32 closed loop, 2 s trot with a lateral push (reading R23): stays within 1e-3 of
    the fp64 oracle's plant trajectory and recovers."""
    N, T = 50, 100
    L = synth.round_to(synth.srbd_problem(2, N + T + 1, seed=1, randomize=False, v_cmd=(0.3, 0.0)), np.float32)
    push = lambda node: np.array([[0.0, 50.0, 0.0]] * 2) if 30 <= node < 36 else None
    r = O.closed_loop(L, N, T, push=push)
    xs, sts = run_gpu_loop(P, L, N, T, torch.float32, 1, push)
    assert np.abs(xs - r["x_plant"]).max() <= 1e-3
    assert (sts[..., 4] == 0).all()
    assert np.abs(xs[:, 86:, 7]).max() < 0.1


def test_closed_loop_batch_tracking_fp32(P):
    """Table-I style: many environments with randomized commands, each with its own MPC; every one
    tracks its commanded velocity over 2 s (mean |v - v_ref| < 0.1 m/s), no failures."""
    B, N, T = 512, 50, 100
    L = synth.srbd_problem(B, N + T + 1, seed=33)
    xs, sts = run_gpu_loop(P, L, N, T, torch.float32)
    assert np.isfinite(xs).all() and (sts[..., 4] == 0).all()
    verr = np.abs(xs[:, 1:, 6:8] - L["x_ref"][:, 1:T + 1, 6:8]).mean(axis=(1, 2))
    assert verr.max() < 0.1, (verr.max(), int(verr.argmax()))


def test_closed_loop_horizon_exhausted(P):
    N = 10
    L = synth.srbd_problem(2, N + 3, seed=2)
    B = 2
    h = handle(P, B, N, torch.float32, L["params"])
    ref = {k: dev(L[k], torch.float32) for k in ("x_ref", "u_ref", "contact", "feet")}
    it0 = {"x": dev(L["x"][:, :N + 2], torch.float32), "u": dev(L["u"][:, :N + 1], torch.float32),
           "lam": dev(L["lam"][:, :N + 2], torch.float32)}
    cl = P.ClosedLoop(h, ref, it0, dev(L["x0"], torch.float32))
    for _ in range(3):
        cl.tick()
    with pytest.raises(RuntimeError):
        cl.tick()
