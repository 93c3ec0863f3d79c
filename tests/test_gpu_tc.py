"""The tcgen05 3xTF32 product used by the large-n fold (tc.cuh, K7), in isolation through
pdilqr_debug_tc_gemm: against an fp64 matmul of the same fp32 inputs, every transpose
combination, ragged shapes (M, N, K not multiples of the 128 x 16 x 16 tiles), one and two M
tiles and N tiles, with and without Cin.  3xTF32 keeps about 2^-19 of relative accuracy per
product, so the error bound is 1e-5 of sum_k |a_ik||b_kj| (plain TF32 would be ~1e-3)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_07823_b200 as P
    P.lib()
    return P


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("M,N,K", [(128, 128, 16), (74, 74, 74), (74, 32, 74), (32, 74, 74), (192, 192, 192),
                                   (200, 130, 37), (1, 8, 3), (256, 256, 64)])
def test_tc_gemm_matches_fp64(P, ta, tb, M, N, K):
    from paper_2506_07823_b200.pdilqr import debug_tc_gemm
    g = torch.Generator(device="cuda").manual_seed(M * 1000 + N * 10 + K)
    A = torch.randn((K, M) if ta else (M, K), device="cuda", generator=g)
    B = torch.randn((N, K) if tb else (K, N), device="cuda", generator=g)
    Cin = torch.randn(M, N, device="cuda", generator=g)
    C = debug_tc_gemm(A, B, Cin, ta, tb)
    torch.cuda.synchronize()
    Ad = (A.T if ta else A).double(); Bd = (B.T if tb else B).double()
    ref = Cin.double() + Ad @ Bd
    scale = Ad.abs() @ Bd.abs() + Cin.double().abs()
    err = ((C.double() - ref).abs() / scale).max().item()
    assert err <= 1e-5, err
    C0 = debug_tc_gemm(A, B, None, ta, tb)
    err0 = ((C0.double() - (Ad @ Bd)).abs() / (Ad.abs() @ Bd.abs())).max().item()
    assert err0 <= 1e-5, err0
