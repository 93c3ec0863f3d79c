"""GPU parity of the centralized multi-robot model (NEXT-3; config 4 of SURVEY §8(d)): the dense
linearisation (k_multi_linearize) against oracle_multi_linearize, and one SQP step (linearise ->
large-n LQ solve -> multi-robot filter line search -> update) against oracle_multi_step, on
identical seeded, dtype-rounded inputs; config 4 itself (16 robots, n = m = 192, N = 50)."""
import numpy as np
import pytest
import torch

from tests import kkt_dense
from tests.gpu_util import rel, rounded, to_device, to_np
from workloads import synth

pytestmark = pytest.mark.gpu
KEYS = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def problem(B, R, N, seed, dtype, spacing=1.0, perturb=0.0):
    p = synth.multi_srbd_problem(B, R, N=N, seed=seed, spacing=spacing)
    if perturb:
        rng = np.random.default_rng(seed)
        p["lam"] = perturb * rng.standard_normal(p["lam"].shape)
        p["u"] = p["u"] + perturb * rng.standard_normal(p["u"].shape)
    return rounded(p, dtype)


def handle(P, p, dtype, B, R, N):
    return P.PdIlqr(N=N, n=12 * R, m=12 * R, batch=B, dtype=dtype, model="multi_srbd", srbd=p["params"],
                    multi=p["multi"])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("R", [1, 2, 5])
def test_multi_linearize_parity(P, O, dtype, R):
    B, N = 2, 7
    p = problem(B, R, N, 11 + R, dtype, spacing=0.8, perturb=1.0)
    h = handle(P, p, dtype, B, R, N)
    out = h.linearize(to_device({k: p[k] for k in KEYS}, dtype))
    torch.cuda.synchronize()
    assert (to_np(out["info"]) == 0).all()
    tol = 2e-5 if dtype == torch.float32 else 1e-11
    for b in range(B):
        ref = O.multi_linearize_single(p, b)
        assert ref["info"] == 0
        for k in ("A", "Bm", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0"):
            g = to_np(out[k][b])
            assert np.abs(g - ref[k]).max() <= tol * max(1.0, np.abs(ref[k]).max()), (k, b)
        assert np.abs(to_np(out["c"][b]) - ref["c"]).max() <= tol * max(1.0, np.abs(p["x"]).max())


def step_parity(P, O, B, R, N, dtype, seed, spacing=1.0, sample=None, tol=None):
    p = problem(B, R, N, seed, dtype, spacing=spacing)
    h = handle(P, p, dtype, B, R, N)
    dev = to_device({k: p[k] for k in KEYS}, dtype)
    d = h.new_direction()
    st = h.step(dev, direction=d)
    torch.cuda.synchronize()
    tol = tol or (1e-4 if dtype == torch.float32 else 1e-9)
    worst = 0.0
    for b in (range(B) if sample is None else sample):
        x, u, lam, st_r, dx, du, dl = O.multi_step_single(p, b)
        assert st_r[4] == 0 and int(to_np(st["info"])[b]) == 0
        lin = O.multi_linearize_single(p, b)
        qp = {k: v[None] for k, v in lin.items() if k != "info"}
        eta = kkt_dense.backward_error_blockwise(qp, 0, to_np(d["dx"][b]), to_np(d["du"][b]), to_np(d["dlam"][b]))
        assert eta <= (1e-5 if dtype == torch.float32 else 1e-12), eta
        for k, ref in (("dx", dx), ("du", du), ("dlam", dl)):
            e = rel(to_np(d[k][b]), ref)
            worst = max(worst, e)
            assert e <= tol, (k, b, e)
        assert float(to_np(st["alpha"])[b]) == st_r[2], (b, float(to_np(st["alpha"])[b]), st_r[2])
        for k, ref in (("x", x), ("u", u), ("lam", lam)):
            e = rel(to_np(dev[k][b]) - p[k][b], ref - p[k][b])
            assert e <= tol, (k, b, e)
        assert abs(float(to_np(st["cost"])[b]) - st_r[0]) <= 10 * tol * max(1.0, abs(st_r[0]))
        assert abs(float(to_np(st["theta"])[b]) - st_r[1]) <= 10 * tol * max(1.0, abs(st_r[1]))
    return worst


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("R,N,B", [(1, 10, 2), (2, 12, 3), (4, 20, 2), (2, 0, 2), (3, 1, 1)])
def test_multi_step_parity(P, O, dtype, R, N, B):
    step_parity(P, O, B, R, N, dtype, seed=20 + R, spacing=0.9)


def test_config4_sixteen_robots(P, O):
    """Config 4: 16 robots on a 4 x 4 grid 1.5 m apart, n = m = 192, N = 50, B = 1,
    fp32, one full SQP step through the large-n path."""
    step_parity(P, O, 1, 16, 50, torch.float32, seed=44, spacing=1.5)


def test_config4_batch_sampled(P, O):
    """Config 4 at B = 8 (cluster size 8 per instance), two instances checked."""
    step_parity(P, O, 8, 16, 50, torch.float32, seed=45, spacing=1.5, sample=[0, 7])
