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


@pytest.fixture(autouse=True, params=["simt", "tc", "mma"])
def products(request, monkeypatch):
    """Every large-path test runs with the SIMT FP32 products, the tcgen05 3xTF32 products
    (PDILQR_BIG_TC=1; tc.cuh) and the warp-level mma.sync 3xTF32 products (PDILQR_BIG_MMA=1;
    big_ric.cuh mma_gemm) of k_big_ric -- the same parity bar for all three."""
    monkeypatch.setenv("PDILQR_BIG_TC", "1" if request.param == "tc" else "0")
    monkeypatch.setenv("PDILQR_BIG_MMA", "1" if request.param == "mma" else "0")
    return request.param


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
        assert np.abs(out["K"][b] - r["K"]).max() <= 1e-4 * max(1.0, np.abs(r["K"]).max())


def test_big_info(P):
    qp = synth.random_lq(2, 5, 20, 8, seed=1)
    qp["R"][1, 2] = -np.eye(8)
    out = solve(P, qp, torch.float32)
    assert out["info"][0] == 0 and out["info"][1] == 3


@pytest.mark.parametrize("B", [1, 5, 40, 160])
def test_cluster_sizes(P, O, B):
    """k_big_ric with one CTA per instance (B >= 74: cluster size 1, config-5 tile shape) and with
    clusters of 2..16 CTAs per instance (small B): same parity on a ragged size (n = 38, m = 21)."""
    qp = rounded(synth.random_lq(B, 6, 38, 21, kind="wb" if B % 2 else "dense", seed=B), torch.float32)
    out = solve(P, qp, torch.float32)
    check(O, qp, out, 1e-4)


def test_config5_tile_shape_batch(P, O):
    """Config-5 dimensions at B = 148 (cluster size 1, 80 x 32 tiles) on 2 distinct instances tiled."""
    base = rounded(synth.random_lq(2, 12, 74, 32, kind="wb", seed=5), torch.float32)
    qp = {k: np.concatenate([v] * 74, axis=0) for k, v in base.items()}
    out = solve(P, qp, torch.float32)
    ref = O.solve_lq({k: v[:2] for k, v in qp.items()})
    for k in ("dx", "du", "dlam"):
        for b in (0, 1, 146, 147):
            r = rel_per_instance(out[k][b:b + 1], ref[k][b % 2:b % 2 + 1])
            assert r.max() <= 1e-4, (k, b, r.max())


def test_legacy_matches_fused(P, monkeypatch):
    """The element/fold/policy kernels (PDILQR_BIG_LEGACY=1, the M-solve combine) and the fused
    Riccati-form kernel agree (both are the same KKT solution, D7)."""
    qp = rounded(synth.random_lq(3, 10, 24, 18, seed=11), torch.float32)
    a = solve(P, qp, torch.float32)
    monkeypatch.setenv("PDILQR_BIG_LEGACY", "1")
    b = solve(P, qp, torch.float32)
    for k in ("dx", "du", "dlam"):
        assert rel_per_instance(a[k], b[k]).max() <= 1e-4, k
