"""GPU parity of the paper's reverse associative scan on the large-dimension path (16 < max(n, m)
<= 256): a handle created with leaf_chunk = 1 runs the Kogge-Stone tree of full combines (Eq. 11,
readings R1-R3; k_bigks_level) instead of the sequential Riccati-form fold, then the stage-parallel
policy and the rollout -- against the fp64 oracle's sequential Riccati solve."""
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


def solve_tree(P, qp, dtype):
    B, N1, n, _ = qp["A"].shape
    m = qp["Bm"].shape[-1]
    h = P.PdIlqr(N=N1 - 1, n=n, m=m, batch=B, dtype=dtype, leaf_chunk=1)
    out = h.solve_lq(to_device(qp, dtype), policy=True)
    torch.cuda.synchronize()
    return {k: to_np(v) for k, v in out.items()}, h.last_launch_count()


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.float64, 1e-9)])
@pytest.mark.parametrize("dims", [(20, 5, 9, 3, "dense"), (33, 40, 12, 2, "dense"), (74, 32, 20, 2, "wb"),
                                  (192, 192, 6, 1, "dense")])
def test_tree_scan_large(P, O, dtype, tol, dims):
    n, m, N, B, kind = dims
    qp = rounded(synth.random_lq(B, N, n, m, kind=kind, seed=90 + n), dtype)
    out, launches = solve_tree(P, qp, dtype)
    ref = O.solve_lq(qp)
    assert (ref["info"] == 0).all() and (out["info"] == 0).all(), out["info"]
    for k in ("dx", "du", "dlam"):
        r = rel_per_instance(out[k], ref[k])
        assert r.max() <= tol, (k, r.max())
    eta = kkt_dense.backward_error_blockwise(qp, 0, out["dx"][0], out["du"][0], out["dlam"][0])
    assert eta <= (1e-5 if dtype == torch.float32 else 1e-12)
    # ceil(log2(N + 2)) Kogge-Stone levels + read-out + init + policy + rollout (+ info)
    assert launches >= int(np.ceil(np.log2(N + 2))) + 4
