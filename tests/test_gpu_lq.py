"""GPU parity of pdilqr_solve_lq (element init -> reverse scan -> policy -> forward scan -> dual
update, all in libpdilqr.so) against the fp64 oracle (sequential Riccati) on identical seeded,
dtype-rounded inputs.  Tolerances (north_star): f32 rel <= 1e-4 on dx, du, dlam
per instance and KKT backward error eta <= 1e-5; f64 rel <= 1e-9."""
import numpy as np
import pytest
import torch

from tests import kkt_dense
from tests.gpu_util import rel, rel_per_instance, rounded, to_device, to_np
from workloads import synth

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.float64: 1e-9}


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def run_gpu(P, qp, dtype, leaf_chunk=0, policy=True):
    B, N1, n, _ = qp["A"].shape
    m = qp["Bm"].shape[-1]
    h = P.PdIlqr(N=N1 - 1, n=n, m=m, batch=B, dtype=dtype, leaf_chunk=leaf_chunk)
    out = h.solve_lq(to_device(qp, dtype), policy=policy)
    torch.cuda.synchronize()
    return {k: to_np(v) for k, v in out.items()}, h


def check(O, qp, dtype, out, kkt=True):
    ref = O.solve_lq(qp)
    assert (ref["info"] == 0).all()
    assert (out["info"] == 0).all(), out["info"]
    for k in ("dx", "du", "dlam"):
        r = rel_per_instance(out[k], ref[k])
        assert r.max() <= TOL[dtype], (k, r.max(), int(r.argmax()))
    if kkt:
        for b in range(min(qp["A"].shape[0], 8)):
            eta = kkt_dense.backward_error_blockwise(qp, b, out["dx"][b], out["du"][b], out["dlam"][b])
            assert eta <= (1e-5 if dtype == torch.float32 else 1e-12), (b, eta)
    return ref


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("chunk", [0, 1, 3, 34])
def test_config1_double_integrator(P, O, dtype, chunk):
    qp = rounded(synth.double_integrator(32, variant="kkt"), dtype)
    out, _ = run_gpu(P, qp, dtype, chunk)
    check(O, qp, dtype, out)
    dx, du, lam = kkt_dense.solve(qp)
    assert rel(out["dx"][0], dx) <= TOL[dtype] and rel(out["dlam"][0], lam) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_config1_dare_fixed_point(P, O, dtype):
    import scipy.linalg as sla
    qp = synth.double_integrator(32, variant="dare")
    A, Bm, Q, R = qp["A"][0, 0], qp["Bm"][0, 0], qp["Q"][0, 0], qp["R"][0, 0]
    qp["P_term"] = sla.solve_discrete_are(A, Bm, Q, R)[None].copy()
    qp = rounded(qp, dtype)
    Kinf = -np.linalg.solve(qp["R"][0, 0] + qp["Bm"][0, 0].T @ qp["P_term"][0] @ qp["Bm"][0, 0],
                            qp["Bm"][0, 0].T @ qp["P_term"][0] @ qp["A"][0, 0])
    out, _ = run_gpu(P, qp, dtype, 1)
    for i in range(33):
        assert rel(out["K"][0, i], Kinf) <= (1e-4 if dtype == torch.float32 else 1e-9)
    check(O, qp, dtype, out)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("chunk", [1, 4, 7, 52])
def test_random_dense_12x12(P, O, dtype, chunk):
    qp = rounded(synth.random_lq(37, 50, 12, 12, seed=101), dtype)
    out, _ = run_gpu(P, qp, dtype, chunk)
    ref = check(O, qp, dtype, out)
    # the policy K, k also matches the oracle's Riccati gains
    for b in (0, 17, 36):
        r1 = O.solve_lq_single(qp, b)
        assert rel(out["K"][b], r1["K"]) <= TOL[dtype]
        assert rel(out["k"][b], r1["k"]) <= TOL[dtype]
    assert ref is not None


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("N", [0, 1, 50])
def test_elem_init_two_rows_per_lane(P, O, monkeypatch, dtype, N):
    """The opt-in two-rows-per-lane element initialisation (PDILQR_ELEM_R2=1, k_elem_init_r2):
    B = 37 (partial warps: shadow workers store nothing), terminal items in every warp mix."""
    monkeypatch.setenv("PDILQR_ELEM_R2", "1")
    qp = rounded(synth.random_lq(37, N, 12, 12, seed=111 + N), dtype)
    out, _ = run_gpu(P, qp, dtype, N + 2)
    check(O, qp, dtype, out)


@pytest.mark.parametrize("dims", [(3, 2, 9), (5, 1, 17), (8, 4, 30), (8, 8, 11), (16, 16, 20), (13, 7, 25), (1, 1, 5)])
@pytest.mark.parametrize("chunk", [1, 5, 0])
def test_padded_dimensions(P, O, dims, chunk):
    n, m, N = dims
    qp = rounded(synth.random_lq(5, N, n, m, seed=7 + n), torch.float32)
    out, _ = run_gpu(P, qp, torch.float32, chunk)
    check(O, qp, torch.float32, out)


@pytest.mark.parametrize("N", [0, 1, 2, 6, 63, 64, 65])
@pytest.mark.parametrize("chunk", [1, 2, 0])
def test_horizon_edges(P, O, N, chunk):
    qp = rounded(synth.random_lq(3, N, 12, 12, seed=N), torch.float32)
    out, _ = run_gpu(P, qp, torch.float32, chunk)
    check(O, qp, torch.float32, out)


def test_wb_sized_problem_structure(P, O):
    """config-5 recipe (second-order structure, diagonal Q/R, 1% time variation) at n=16 m=8."""
    qp = rounded(synth.random_lq(8, 100, 16, 8, kind="wb"), torch.float32)
    out, _ = run_gpu(P, qp, torch.float32, 0)
    check(O, qp, torch.float32, out)


@pytest.mark.parametrize("N", [200, 1000])
def test_long_horizon_tree(P, O, N):
    qp = rounded(synth.random_lq(2, N, 12, 12, seed=N), torch.float32)
    out, _ = run_gpu(P, qp, torch.float32, 1)
    check(O, qp, torch.float32, out, kkt=False)


def test_full_batch_4096_sampled(P, O):
    """BASELINE config-3 size (B=4096, N=50, n=m=12) in the launch configuration bench.py times;
    a sample of instances (first, last, random) is checked against the oracle one by one."""
    qp = rounded(synth.random_lq(4096, 50, 12, 12, seed=5), torch.float32)
    out, _ = run_gpu(P, qp, torch.float32, 0, policy=False)
    assert (out["info"] == 0).all()
    idx = [0, 1, 4095] + list(np.random.default_rng(0).choice(4096, 13, replace=False))
    for b in idx:
        r = O.solve_lq_single(qp, b)
        for k in ("dx", "du", "dlam"):
            assert rel(out[k][b], r[k]) <= 1e-4, (b, k)


def test_bitwise_deterministic(P):
    qp = rounded(synth.random_lq(64, 50, 12, 12, seed=9), torch.float32)
    h = P.PdIlqr(N=50, n=12, m=12, batch=64, dtype=torch.float32, leaf_chunk=4)
    d = to_device(qp, torch.float32)
    a = h.solve_lq(d)
    a = {k: v.clone() for k, v in a.items()}
    b = h.solve_lq(d)
    torch.cuda.synchronize()
    for k in ("dx", "du", "dlam"):
        assert torch.equal(a[k], b[k])


def test_info_reports_failing_stage(P):
    qp = synth.random_lq(4, 10, 12, 12, seed=3)
    qp["R"][2, 3] = -np.eye(12)      # R_3 of instance 2 not positive definite
    qp["dx0"][1, 0] = np.nan          # instance 1: non-finite data
    out, _ = run_gpu(P, qp, torch.float32, 0)
    assert out["info"][0] == 0 and out["info"][3] == 0
    assert out["info"][2] == 4
    assert out["info"][1] == -1


def test_rejects_bad_arguments(P):
    h = P.PdIlqr(N=5, n=4, m=2, batch=2, dtype=torch.float32)
    qp = to_device(synth.random_lq(2, 5, 4, 2), torch.float32)
    qp["A"] = qp["A"].double()
    with pytest.raises(P.PdilqrError):
        h.solve_lq(qp)
    with pytest.raises(P.PdilqrError):
        P.PdIlqr(N=5, n=300, m=2, batch=2)


@pytest.mark.parametrize("ks", ["0", "1"])
@pytest.mark.parametrize("N", [0, 1, 6, 50, 63, 64, 200])
def test_latency_scan_algorithms(P, O, monkeypatch, ks, N):
    """Latency regime (leaf chunk 1, cooperative grid kernels): the depth-optimal Kogge-Stone reverse
    scan (PDILQR_SCAN_KS=1, default when a level fits in one wave) and the Blelloch tree (=0) both
    match the oracle, across horizons around powers of two."""
    monkeypatch.setenv("PDILQR_SCAN_KS", ks)
    qp = rounded(synth.random_lq(2, N, 12, 12, seed=300 + N), torch.float32)
    out, _ = run_gpu(P, qp, torch.float32, 1)
    check(O, qp, torch.float32, out)


@pytest.mark.parametrize("ks", ["0", "1"])
def test_latency_scan_algorithms_f64_padded(P, O, monkeypatch, ks):
    monkeypatch.setenv("PDILQR_SCAN_KS", ks)
    qp = rounded(synth.random_lq(3, 40, 7, 5, seed=77), torch.float64)
    out, _ = run_gpu(P, qp, torch.float64, 1)
    check(O, qp, torch.float64, out)
