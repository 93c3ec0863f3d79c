"""GPU parity of the large-dimension path (16 < max(n, m) <= 256: BASELINE configs 4 and 5) of
pdilqr_solve_lq against the fp64 oracle on identical seeded, dtype-rounded inputs."""
import numpy as np
import pytest
import torch

from tests import kkt_dense
from tests.gpu_util import rel_per_instance, rounded, to_device, to_np
from workloads import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def solve(P, qp, dtype):
    B, N1, n, _ = qp["A"].shape
    m = qp["Bm"].shape[-1]
    h = P.PdIlqr(N=N1 - 1, n=n, m=m, batch=B, dtype=dtype)
    out = h.solve_lq(to_device(qp, dtype), policy=True)
    torch.cuda.synchronize()
    return {k: to_np(v) for k, v in out.items()}


def check(O, qp, out, tol):
    ref = O.solve_lq(qp)
    assert (ref["info"] == 0).all() and (out["info"] == 0).all(), out["info"]
    worst = {}
    for k in ("dx", "du", "dlam"):
        r = rel_per_instance(out[k], ref[k])
        worst[k] = float(r.max())
        assert r.max() <= tol, (k, r.max())
    return worst


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.float64, 1e-9)])
def test_config5_wb_sized(P, O, dtype, tol):
    """Config 5: whole-body-sized LQ n=74, m=32, N=100 (recipe of SURVEY §8(d)), B=3."""
    qp = rounded(synth.random_lq(3, 100, 74, 32, kind="wb", seed=55), dtype)
    out = solve(P, qp, dtype)
    check(O, qp, out, tol)
    eta = kkt_dense.backward_error_blockwise(qp, 0, out["dx"][0], out["du"][0], out["dlam"][0])
    assert eta <= (1e-5 if dtype == torch.float32 else 1e-12)


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.float64, 1e-9)])
def test_config4_centralized_sized(P, O, dtype, tol):
    """Config 4 dimensions: n = m = 192, N = 50, single instance (dense random data)."""
    qp = rounded(synth.random_lq(1, 50, 192, 192, kind="dense", seed=44), dtype)
    out = solve(P, qp, dtype)
    check(O, qp, out, tol)


@pytest.mark.parametrize("dims", [(17, 5, 9), (33, 40, 12), (64, 16, 20), (20, 20, 0)])
def test_odd_dimensions(P, O, dims):
    n, m, N = dims
    qp = rounded(synth.random_lq(2, N, n, m, seed=n + m), torch.float32)
    out = solve(P, qp, torch.float32)
    check(O, qp, out, 1e-4)
    for b in range(2):
        r = O.solve_lq_single(qp, b)
        assert np.abs(out["K"][b] - r["K"]).max() <= 1e-3 * max(1.0, np.abs(r["K"]).max())


def test_big_info(P):
    qp = synth.random_lq(2, 5, 20, 8, seed=1)
    qp["R"][1, 2] = -np.eye(8)
    out = solve(P, qp, torch.float32)
    assert out["info"][0] == 0 and out["info"][1] == 3
