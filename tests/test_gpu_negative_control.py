"""Negative control: with PDILQR_FAULT_COMBINE=1 the library corrupts one scan element
of instance 0 (P~[0][0] of stage N/2 by 1e-3 relative); the same parity check the LQ tests use must
then fail for instance 0 and still pass for the untouched instance 1 -- the tests can see a wrong
combine.  Without the flag both pass."""
import numpy as np
import pytest
import torch

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


@pytest.mark.parametrize("chunk", [0, 1, 52])
def test_corrupted_combine_turns_parity_red(P, O, monkeypatch, chunk):
    qp = rounded(synth.random_lq(2, 50, 12, 12, seed=3), torch.float64)
    ref = O.solve_lq(qp)

    def worst():
        h = P.PdIlqr(N=50, n=12, m=12, batch=2, dtype=torch.float64, leaf_chunk=chunk)
        out = h.solve_lq(to_device(qp, torch.float64))
        torch.cuda.synchronize()
        return np.max(np.stack([rel_per_instance(to_np(out[k]), ref[k]) for k in ("dx", "du", "dlam")]), axis=0)

    ok = worst()
    assert (ok <= 1e-9).all()
    monkeypatch.setenv("PDILQR_FAULT_COMBINE", "1")
    bad = worst()
    assert bad[0] > 1e-6 and bad[1] <= 1e-9, bad
