// big_ric.cuh -- large-dimension path (16 < max(n, m) <= 256, configs 4 and 5 of SURVEY §8(d)),
// single-chunk schedule with the element, the cheap combine and the policy fused per stage
// (design D7 of DESIGN.md applied to general Eq. 4 data, S != 0):
//
//   s_{N+1} = (P_{N+1}, p_{N+1});  for i = N..0, with (P', p') = (P_{i+1}, p_{i+1}):
//     PB = P' B,  g = p' + P' c                                   (phase 1)
//     G = R + B^T PB,  H = S + PB^T A,  h = r + B^T g             (phase 2)
//     [K | k] = -G^-1 [H | h]   (Cholesky of G, SPD)              (phase 3, Eq. 5 rows)
//     Abar = A + B K,  bbar = c + B k                             (phase 4, Eq. 14)
//     V = P' Abar,  w = p' + P' bbar                              (phase 5)
//     P_i = Q + A^T V + S^T K (re-symmetrised, R22),
//     p_i = q + A^T w + S^T k                                     (phases 6, 7)
//
// This is Eq. 11's cheap combine e_i (x) s_{i+1} (suffix with A~ = C~ = b~ = 0, R1/R5) with the
// element of Eq. 12 substituted and X = (I + C~_i P')^-1 A~_i taken as Abar_i by Woodbury (D7):
// identical in exact arithmetic, no R^-1 and no pivoted n x n elimination.  R is still required
// SPD by Eq. 12: k_big_rchk factorises every R_i in parallel and reports failures with the
// same info code as the element initialisation.
//
// Parallel decomposition: one thread-block cluster of CS CTAs per instance (CS = 16 at B = 1, 1
// when the batch fills the GPU).  Products are distributed over the cluster's CTAs tile by tile
// (16*TM square tiles, TM x TM register micro-tiles, 16-deep k panels staged through shared
// memory, next panel prefetched into registers); matrices live in global memory (L2-resident per
// instance); phases are separated by cluster barriers (release/acquire at cluster scope), operands
// written by another CTA are read with ld.global.cg.  The m x m Cholesky is done redundantly by
// every CTA of the cluster in its own shared memory (no broadcast, no extra barrier); the n + 1
// right-hand sides are split over the cluster's warps, two columns per warp, forward and backward
// substitution warp-synchronously with the factor in shared memory.
#pragma once

#include <cooperative_groups.h>

#include "big.cuh"
#include "tc.cuh"

namespace pdilqr {

constexpr int RIC_THREADS = 256;

template <typename T, int TM>
struct RicTiles {
    T As[16][16 * TM + 1];
    T Bs[16][16 * TM + 1];
};

template <typename T>
__device__ __forceinline__ T ldg_cg(const T *p) { return __ldcg(p); }

__device__ __forceinline__ void ric_sync(int CS) {
    if (CS > 1) cooperative_groups::this_cluster().sync();
    else __syncthreads();
}

// Tiles t = part, part + nparts, ... of C[Mr x Nc] = (Cin ? Cin : 0) + alpha op(A)[Mr x K] op(B)[K x Nc]
// with (16 TR) x (16 TC) output tiles, TR x TC register micro-tiles (rows ty + 16 q, columns
// tx + 16 w: broadcast A reads, conflict-free B reads), 16-deep k panels staged through shared
// memory, the next panel prefetched into registers.  op(A) = A (row-major Mr x K, ld lda) or A^T (A
// stored K x Mr); same for B.  Cin may alias C with the same leading dimension (each element is read
// and written by the same thread).  TR, TC <= TM of the shared tile buffer.
template <typename T, int TR, int TC, bool TA, bool TB, int TM>
__device__ void ric_gemm(int Mr, int Nc, int K, T alpha, const T *A, int lda, const T *Bm, int ldb, const T *Cin,
                         int ldci, T *C, int ldc, int part, int nparts, RicTiles<T, TM> &sm) {
    static_assert(TR <= TM && TC <= TM, "tile buffer too small");
    constexpr int TSR = 16 * TR, TSC = 16 * TC;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int tmn = (Mr + TSR - 1) / TSR, tnn = (Nc + TSC - 1) / TSC;
    // fixed per-thread panel coordinates: element e = tid + 256 s of the 16 x TSR (A) / 16 x TSC (B) panel
    int amm[TR], akk[TR], bnn[TC], bkk[TC];
#pragma unroll
    for (int s = 0; s < TR; ++s) {
        const int e = tid + RIC_THREADS * s;
        if (TA) { amm[s] = e % TSR; akk[s] = e / TSR; } else { akk[s] = e & 15; amm[s] = e >> 4; }
    }
#pragma unroll
    for (int s = 0; s < TC; ++s) {
        const int e = tid + RIC_THREADS * s;
        if (TB) { bkk[s] = e & 15; bnn[s] = e >> 4; } else { bnn[s] = e % TSC; bkk[s] = e / TSC; }
    }
    for (int t = part; t < tmn * tnn; t += nparts) {
        const int tm = (t / tnn) * TSR, tn = (t % tnn) * TSC;
        T acc[TR][TC];
#pragma unroll
        for (int a = 0; a < TR; ++a)
#pragma unroll
            for (int c = 0; c < TC; ++c) acc[a][c] = T(0);
        T pa[TR], pb[TC];
        auto fetch = [&](int k0) {
#pragma unroll
            for (int s = 0; s < TR; ++s) {
                const int r = tm + amm[s], c = k0 + akk[s];
                pa[s] = (r < Mr && c < K) ? ldg_cg(TA ? A + (size_t)c * lda + r : A + (size_t)r * lda + c) : T(0);
            }
#pragma unroll
            for (int s = 0; s < TC; ++s) {
                const int rb = k0 + bkk[s], cb = tn + bnn[s];
                pb[s] = (rb < K && cb < Nc) ? ldg_cg(TB ? Bm + (size_t)cb * ldb + rb : Bm + (size_t)rb * ldb + cb) : T(0);
            }
        };
        fetch(0);
        for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
            for (int s = 0; s < TR; ++s) sm.As[akk[s]][amm[s]] = pa[s];
#pragma unroll
            for (int s = 0; s < TC; ++s) sm.Bs[bkk[s]][bnn[s]] = pb[s];
            __syncthreads();
            if (k0 + 16 < K) fetch(k0 + 16);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                T a[TR], b[TC];
#pragma unroll
                for (int q = 0; q < TR; ++q) a[q] = sm.As[kk][ty + 16 * q];
#pragma unroll
                for (int q = 0; q < TC; ++q) b[q] = sm.Bs[kk][tx + 16 * q];
#pragma unroll
                for (int q = 0; q < TR; ++q)
#pragma unroll
                    for (int w = 0; w < TC; ++w) acc[q][w] = fma(a[q], b[w], acc[q][w]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < TR; ++q) {
            const int r = tm + ty + 16 * q;
            if (r >= Mr) continue;
            T cin[TC];
#pragma unroll
            for (int w = 0; w < TC; ++w) {
                const int c = tn + tx + 16 * w;
                cin[w] = (Cin && c < Nc) ? ldg_cg(Cin + (size_t)r * ldci + c) : T(0);
            }
#pragma unroll
            for (int w = 0; w < TC; ++w) {
                const int c = tn + tx + 16 * w;
                if (c < Nc) C[(size_t)r * ldc + c] = fma(alpha, acc[q][w], cin[w]);
            }
        }
    }
}

// ---------------------------------------------------------------- warp-level tensor-core products
// mma.sync.m16n8k8 TF32 with FP32 accumulation in the 3xTF32 split (x = hi + lo, hi = rn_tf32(x),
// lo = rn_tf32(x - hi); A B ~ hi hi + hi lo + lo hi, the dropped lo lo and the rounding of lo are
// O(2^-22) relative: FP32-level accuracy).  One warp per (16 MF) x (8 NF) output tile,
// tiles spread over all warps of the cluster; fragments are loaded straight from global memory
// (L2-resident per instance) one k-step ahead, so there is no shared-memory staging and no block
// barrier inside a product.  Same contract as ric_gemm (Cin may alias C).
__device__ __forceinline__ uint32_t f2tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <bool TA, bool TB, int MF, int NF>
__device__ void mma_gemm(int Mr, int Nc, int K, float alpha, const float *A, int lda, const float *Bm, int ldb,
                         const float *Cin, int ldci, float *C, int ldc, int part, int nparts) {
    constexpr int WM = 16 * MF, WN = 8 * NF;
    const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
    const int nw = blockDim.x >> 5;
    const int gw = part * nw + (threadIdx.x >> 5), ngw = nparts * nw;
    const int tmn = (Mr + WM - 1) / WM, tnn = (Nc + WN - 1) / WN;
    auto ldA = [&](int r, int k) -> float {
        return (r < Mr && k < K) ? __ldcg(TA ? A + (size_t)k * lda + r : A + (size_t)r * lda + k) : 0.f;
    };
    auto ldB = [&](int k, int c) -> float {
        return (k < K && c < Nc) ? __ldcg(TB ? Bm + (size_t)c * ldb + k : Bm + (size_t)k * ldb + c) : 0.f;
    };
    for (int t = gw; t < tmn * tnn; t += ngw) {
        const int m0 = (t / tnn) * WM, n0 = (t % tnn) * WN;
        float acc[MF][NF][4];
#pragma unroll
        for (int a = 0; a < MF; ++a)
#pragma unroll
            for (int c = 0; c < NF; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[a][c][e] = 0.f;
        float fa[MF][4], fb[NF][2];
        auto fetch = [&](int k0, float (&xa)[MF][4], float (&xb)[NF][2]) {
#pragma unroll
            for (int a = 0; a < MF; ++a) {
                const int r = m0 + 16 * a + g;
                xa[a][0] = ldA(r, k0 + tg);
                xa[a][1] = ldA(r + 8, k0 + tg);
                xa[a][2] = ldA(r, k0 + tg + 4);
                xa[a][3] = ldA(r + 8, k0 + tg + 4);
            }
#pragma unroll
            for (int c = 0; c < NF; ++c) {
                const int cc = n0 + 8 * c + g;
                xb[c][0] = ldB(k0 + tg, cc);
                xb[c][1] = ldB(k0 + tg + 4, cc);
            }
        };
        fetch(0, fa, fb);
        for (int k0 = 0; k0 < K; k0 += 8) {
            float na[MF][4], nb[NF][2];
            const bool more = k0 + 8 < K;
            if (more) fetch(k0 + 8, na, nb);
            uint32_t ah[MF][4], al[MF][4], bh[NF][2], bl[NF][2];
#pragma unroll
            for (int a = 0; a < MF; ++a)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    ah[a][e] = f2tf32(fa[a][e]);
                    al[a][e] = f2tf32(fa[a][e] - __uint_as_float(ah[a][e]));
                }
#pragma unroll
            for (int c = 0; c < NF; ++c)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    bh[c][e] = f2tf32(fb[c][e]);
                    bl[c][e] = f2tf32(fb[c][e] - __uint_as_float(bh[c][e]));
                }
#pragma unroll
            for (int a = 0; a < MF; ++a)
#pragma unroll
                for (int c = 0; c < NF; ++c) {
                    mma_tf32(acc[a][c], al[a], bh[c]);
                    mma_tf32(acc[a][c], ah[a], bl[c]);
                    mma_tf32(acc[a][c], ah[a], bh[c]);
                }
            if (more) {
#pragma unroll
                for (int a = 0; a < MF; ++a)
#pragma unroll
                    for (int e = 0; e < 4; ++e) fa[a][e] = na[a][e];
#pragma unroll
                for (int c = 0; c < NF; ++c) { fb[c][0] = nb[c][0]; fb[c][1] = nb[c][1]; }
            }
        }
#pragma unroll
        for (int a = 0; a < MF; ++a)
#pragma unroll
            for (int c = 0; c < NF; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = m0 + 16 * a + g + (e >= 2 ? 8 : 0);
                    const int cc = n0 + 8 * c + 2 * tg + (e & 1);
                    if (r < Mr && cc < Nc) {
                        const float cin = Cin ? __ldcg(Cin + (size_t)r * ldci + cc) : 0.f;
                        C[(size_t)r * ldc + cc] = fmaf(alpha, acc[a][c][e], cin);
                    }
                }
    }
}

// The products of k_big_ric: SIMT FP32 tiles (ric_gemm), with UT (float only) tcgen05 tensor cores
// in 3xTF32 (tc_gemm, tc.cuh), with MM (float only) warp-level mma.sync in 3xTF32 (mma_gemm).
// Same contract.
template <typename T, int TR, int TC_, bool TA, bool TB, int TM, bool UT, bool MM = false>
__device__ __forceinline__ void big_gemm(int Mr, int Nc, int K, const T *A, int lda, const T *Bm, int ldb, const T *Cin,
                                         int ldci, T *C, int ldc, int part, int nparts, RicTiles<T, TM> &tiles,
                                         TcSmem *tcs, TcPhase &ph) {
    if constexpr (MM && sizeof(T) == 4) {
        mma_gemm<TA, TB, 1, 4>(Mr, Nc, K, 1.0f, reinterpret_cast<const float *>(A), lda,
                               reinterpret_cast<const float *>(Bm), ldb, reinterpret_cast<const float *>(Cin), ldci,
                               reinterpret_cast<float *>(C), ldc, part, nparts);
    } else if constexpr (UT) {
        tc_gemm<TA, TB>(Mr, Nc, K, 1.0f, A, lda, Bm, ldb, Cin, ldci, C, ldc, part, nparts, *tcs, ph);
    } else {
        ric_gemm<T, TR, TC_, TA, TB, TM>(Mr, Nc, K, T(1), A, lda, Bm, ldb, Cin, ldci, C, ldc, part, nparts, tiles);
    }
}

// Rows r = gw, gw + nw, ... of y = (yin ? yin : 0) + op(A)[Mr x K] x (yin may alias y), y and yin with
// strides incy, inci.  op(A) = A: one warp per four rows (lanes over k, four independent row sums in
// flight); op(A) = A^T: warp gw takes rows 32 gw + lane (coalesced columns of the stored K x Mr
// matrix), k unrolled by 4.
template <typename T, bool TA>
__device__ void ric_gemv(int Mr, int K, const T *A, int lda, const T *x, const T *yin, int inci, T *y, int incy,
                         int gw, int nw) {
    const int lane = threadIdx.x & 31;
    if constexpr (TA) {
        for (int r0 = 32 * gw; r0 < Mr; r0 += 32 * nw) {
            const int r = r0 + lane;
            const bool act = r < Mr;
            const int rc = act ? r : Mr - 1;
            T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
            int k = 0;
            for (; k + 4 <= K; k += 4) {
                s0 = fma(ldg_cg(A + (size_t)k * lda + rc), ldg_cg(x + k), s0);
                s1 = fma(ldg_cg(A + (size_t)(k + 1) * lda + rc), ldg_cg(x + k + 1), s1);
                s2 = fma(ldg_cg(A + (size_t)(k + 2) * lda + rc), ldg_cg(x + k + 2), s2);
                s3 = fma(ldg_cg(A + (size_t)(k + 3) * lda + rc), ldg_cg(x + k + 3), s3);
            }
            for (; k < K; ++k) s0 = fma(ldg_cg(A + (size_t)k * lda + rc), ldg_cg(x + k), s0);
            const T s = (s0 + s1) + (s2 + s3);
            if (act) y[(size_t)r * incy] = yin ? ldg_cg(yin + (size_t)r * inci) + s : s;
        }
    } else {
        for (int r0 = 4 * gw; r0 < Mr; r0 += 4 * nw) {
            T s[4] = {T(0), T(0), T(0), T(0)};
            for (int k = lane; k < K; k += 32) {
                const T xk = ldg_cg(x + k);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (r0 + q < Mr) s[q] = fma(ldg_cg(A + (size_t)(r0 + q) * lda + k), xk, s[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], off);
            }
            if (lane < 4 && r0 + lane < Mr) {
                const int r = r0 + lane;
                const T v = lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3];
                y[(size_t)r * incy] = yin ? ldg_cg(yin + (size_t)r * inci) + v : v;
            }
        }
    }
}

__host__ __device__ constexpr int ric_ldl(int m) { return (m & 1) ? m : m + 1; }  // odd: conflict-free rows and columns

// In-place Cholesky of the m x m SPD matrix in shared memory L (row-major, ld odd so that rows and
// columns are both conflict-free), CTA-wide, any block size (multiple of 32).  Blocked right-looking
// with 16-wide column blocks: (a) the 16 x 16 diagonal block by warp 0 (lane = row, warp-synchronous),
// (b) the panel below it, one thread per row (forward substitution against the diagonal block),
// (c) the trailing update A22 -= L21 L21^T as 64 x 64 register-tiled products (16 x 16 virtual
// threads, 4 x 4 micro-tiles, 16-deep), only tiles on or below the diagonal.  On return the lower
// triangle holds L (the upper triangle is scratch) and dinv[k] = 1/L_kk.  Returns false if a pivot is
// not > 0 and finite (the factor is then garbage).
template <typename T>
__device__ bool cta_chol(int m, T *L, int ld, T *dinv) {
    __shared__ int s_ok;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x;
    if (tid == 0) s_ok = 1;
    for (int kb = 0; kb < m; kb += 16) {
        const int nb = min(16, m - kb);
        if (wid == 0) {  // (a) diagonal block: lane i < nb holds row kb + i in registers
            T x[16];
            const bool own = lane < nb;
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = (own && j < nb) ? L[(size_t)(kb + lane) * ld + kb + j] : T(0);
            bool ok = true;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k < nb) {
                    const T d = __shfl_sync(0xffffffffu, x[k], k);
                    ok = ok && d > T(0) && isfinite(d);
                    const T sd = sqrt(d), is = T(1) / sd;
                    const T lik = lane > k ? x[k] * is : (lane == k ? sd : T(0));
                    x[k] = lane >= k ? lik : x[k];
                    if (lane == 0) dinv[kb + k] = is;
#pragma unroll
                    for (int j = k + 1; j < 16; ++j) {
                        const T ljk = __shfl_sync(0xffffffffu, lik, j);
                        if (lane >= j) x[j] = fma(-lik, ljk, x[j]);
                    }
                }
            }
            if (own) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j <= lane && j < nb) L[(size_t)(kb + lane) * ld + kb + j] = x[j];
            }
            if (!ok && lane == 0) s_ok = 0;
        }
        __syncthreads();
        const int r0 = kb + nb, rem = m - r0;
        if (rem <= 0) break;
        for (int i = r0 + tid; i < m; i += nt) {  // (b) panel: L21 = A21 L11^-T
            T *Li = L + (size_t)i * ld + kb;
            T x[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = j < nb ? Li[j] : T(0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j < nb) {
                    T s = x[j];
                    const T *Lj = L + (size_t)(kb + j) * ld + kb;
#pragma unroll
                    for (int p = 0; p < j; ++p) s = fma(-x[p], Lj[p], s);
                    x[j] = s * dinv[kb + j];
                }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nb) Li[j] = x[j];
        }
        __syncthreads();
        const int nbt = (rem + 63) / 64;  // (c) trailing update, 64 x 64 tiles (ti >= tj)
        for (int v = tid; v < 256 * nbt * (nbt + 1) / 2; v += nt) {
            int t = v >> 8;
            int ti = 0;
            while (t > ti) { t -= ti + 1; ++ti; }
            const int tj = t, tx = v & 15, ty = (v >> 4) & 15;
            T acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] = T(0);
            int ri[4], ci[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ri[q] = min(r0 + ti * 64 + ty + 16 * q, m - 1);
                ci[q] = min(r0 + tj * 64 + tx + 16 * q, m - 1);
            }
            for (int p = 0; p < nb; ++p) {
                T a[4], b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) { a[q] = L[(size_t)ri[q] * ld + kb + p]; b[q] = L[(size_t)ci[q] * ld + kb + p]; }
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int w = 0; w < 4; ++w) acc[q][w] = fma(a[q], b[w], acc[q][w]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = r0 + ti * 64 + ty + 16 * q;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const int c = r0 + tj * 64 + tx + 16 * w;
                    if (r < m && c <= r) L[(size_t)r * ld + c] -= acc[q][w];
                }
            }
        }
        __syncthreads();
    }
    __syncthreads();
    return s_ok != 0;
}

// One warp solves G x = rhs for two right-hand sides with the Cholesky factor in shared memory:
// forward L y = rhs, backward L^T x = y.  Lane l holds rows l + 32 s (s < MS, m <= 32 MS).
template <typename T, int MS>
__device__ void warp_chol_solve2(int m, const T *L, int ld, const T *dinv, T (&b0)[8], T (&b1)[8]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 0; s < MS; ++s) {
#pragma unroll 8
        for (int jj = 0; jj < 32; ++jj) {
            const int j = s * 32 + jj;
            if (j < m) {
                const T dj = dinv[j];
                const T y0 = __shfl_sync(0xffffffffu, b0[s], jj) * dj;
                const T y1 = __shfl_sync(0xffffffffu, b1[s], jj) * dj;
                if (lane == jj) { b0[s] = y0; b1[s] = y1; }
#pragma unroll
                for (int s2 = s; s2 < MS; ++s2) {
                    const int i = s2 * 32 + lane;
                    if (i > j && i < m) {
                        const T l = L[(size_t)i * ld + j];
                        b0[s2] = fma(-l, y0, b0[s2]);
                        b1[s2] = fma(-l, y1, b1[s2]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int s = MS - 1; s >= 0; --s) {
#pragma unroll 8
        for (int jj = 31; jj >= 0; --jj) {
            const int j = s * 32 + jj;
            if (j < m) {
                const T dj = dinv[j];
                const T x0 = __shfl_sync(0xffffffffu, b0[s], jj) * dj;
                const T x1 = __shfl_sync(0xffffffffu, b1[s], jj) * dj;
                if (lane == jj) { b0[s] = x0; b1[s] = x1; }
#pragma unroll
                for (int s2 = 0; s2 <= s; ++s2) {
                    const int i = s2 * 32 + lane;
                    if (i < j) {
                        const T l = L[(size_t)j * ld + i];
                        b0[s2] = fma(-l, x0, b0[s2]);
                        b1[s2] = fma(-l, x1, b1[s2]);
                    }
                }
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ void warp_chol_solve2_any(int m, const T *L, int ld, const T *dinv, T (&b0)[8], T (&b1)[8]) {
    if (m <= 32) warp_chol_solve2<T, 1>(m, L, ld, dinv, b0, b1);
    else if (m <= 64) warp_chol_solve2<T, 2>(m, L, ld, dinv, b0, b1);
    else if (m <= 128) warp_chol_solve2<T, 4>(m, L, ld, dinv, b0, b1);
    else warp_chol_solve2<T, 8>(m, L, ld, dinv, b0, b1);
}

// Copy an m x m row-major matrix (leading dimension lds, global memory) into the shared factor
// buffer (leading dimension ldl): one warp per row, lanes over columns (coalesced, no index
// division), all of a row's loads issued before its stores.
template <typename T>
__device__ __forceinline__ void copy_rows_to_factor(int m, const T *src, int lds, T *Ls, int ldl) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = wid; r < m; r += nw) {
        T v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = lane + 32 * j;
            v[j] = c < m ? ldg_cg(src + (size_t)r * lds + c) : T(0);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = lane + 32 * j;
            if (c < m) Ls[(size_t)r * ldl + c] = v[j];
        }
    }
}

// Per-instance global scratch of k_big_ric (values of T): PB [n x ld(m)], W = [G | H | h]
// [m x ld(m+n+1)], V [n x LD], g, w [LD each].
__host__ __device__ inline size_t ric_slot(int n, int m) {
    return (size_t)n * ld_of(m) + (size_t)m * ld_of(m + n + 1) + (size_t)n * ld_of(n) + 2 * (size_t)ld_of(n);
}

__host__ __device__ inline size_t ric_smem_bytes(int m, int esz) {
    return ((size_t)m * ric_ldl(m) + (size_t)ld_of(m)) * esz;
}

// ... plus the tensor-core panel buffers (128-byte aligned) of the UT variant
__host__ __device__ inline size_t ric_tc_offset(int m, int esz) { return (ric_smem_bytes(m, esz) + 127) / 128 * 128; }
__host__ __device__ inline size_t ric_smem_bytes_tc(int m) { return ric_tc_offset(m, 4) + sizeof(TcSmem); }
constexpr uint32_t RIC_TMEM_COLS = 128;

// Fused reverse scan + policy (phases 1-7 above), one cluster of CS CTAs per instance.
// Writes P_i, p_i (ws.Pp), K_i, k_i (ws.Kk, out.K, out.k), Abar_i, bbar_i (ws.tel).
template <typename T, int TN, int TU, bool UT = false, bool MM = false>
__global__ void __launch_bounds__(RIC_THREADS, 2) k_big_ric(LqArgs<T> qp, int B, int N, BigDims<T> d, BigWork<T> ws,
                                                         LqOut<T> out, int CS) {
    static_assert(!UT || sizeof(T) == 4, "tensor-core products are FP32 (3xTF32) only");
    static_assert(!MM || sizeof(T) == 4, "mma.sync products are FP32 (3xTF32) only");
    constexpr int TM = (UT || MM) ? 1 : (TN > TU ? TN : TU);
    __shared__ RicTiles<T, TM> tiles;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = d.n, m = d.m, LD = d.LD, LDU = d.LDU;
    const int b = blockIdx.x / CS, rank = blockIdx.x % CS;
    if (b >= B) return;  // whole clusters only (grid = B * CS)
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nwl = RIC_THREADS / 32;
    const int gw = rank * nwl + wid, nwc = CS * nwl;
    const int ldpb = ld_of(m), ldw = ld_of(m + n + 1), ldl = ric_ldl(m);
    T *Ls = reinterpret_cast<T *>(dyn), *dinv = Ls + (size_t)m * ldl;
    T *PB = ws.scratch + (size_t)b * ws.slot, *W = PB + (size_t)n * ldpb, *V = W + (size_t)m * ldw,
      *g = V + (size_t)n * LD, *w = g + LD;
    T *Pp = ws.Pp + (size_t)b * (N + 2) * d.psize();
    TcSmem *tcs = nullptr;
    TcPhase ph;
    if constexpr (UT) {
        tcs = reinterpret_cast<TcSmem *>(dyn + ric_tc_offset(m, sizeof(T)));
        tc_alloc(*tcs, RIC_TMEM_COLS);
    }
    {   // s_{N+1} = (P_{N+1}, p_{N+1})
        T *Pt = Pp + (size_t)(N + 1) * d.psize();
        for (int t = rank * RIC_THREADS + threadIdx.x; t < n * n; t += CS * RIC_THREADS)
            Pt[(size_t)(t / n) * LD + t % n] = qp.Pt[(size_t)b * n * n + t];
        for (int t = rank * RIC_THREADS + threadIdx.x; t < n; t += CS * RIC_THREADS)
            Pt[(size_t)n * LD + t] = qp.pt[(size_t)b * n + t];
    }
    ric_sync(CS);
    int fail = INT_MAX;
    for (int i = N; i >= 0; --i) {
        const size_t st = (size_t)b * (N + 1) + i;
        const T *A = qp.A + st * n * n, *Bm = qp.Bm + st * n * m, *R = qp.R + st * m * m;
        const T *S = qp.S ? qp.S + st * m * n : nullptr, *q = qp.q + st * n, *r = qp.r + st * m, *c = qp.c + st * n;
        const T *Pn = Pp + (size_t)(i + 1) * d.psize(), *pn = Pn + (size_t)n * LD;
        T *Pc = Pp + (size_t)i * d.psize(), *pc = Pc + (size_t)n * LD;
        T *Kw = ws.Kk + st * d.ksize(), *kw = Kw + (size_t)m * LD;
        T *Ab = ws.tel + st * d.psize(), *bb = Ab + (size_t)n * LD;
        // phase 1: PB = P' B ; g = p' + P' c
        big_gemm<T, TN, TU, false, false, TM, UT, MM>(n, m, n, Pn, LD, Bm, m, nullptr, 0, PB, ldpb, rank, CS, tiles, tcs, ph);
        ric_gemv<T, false>(n, n, Pn, LD, c, pn, 1, g, 1, gw, nwc);
        ric_sync(CS);
        // phase 2: W = [R + B^T PB | S + PB^T A | r + B^T g]
        big_gemm<T, TU, TU, true, false, TM, UT, MM>(m, m, n, Bm, m, PB, ldpb, R, m, W, ldw, rank, CS, tiles, tcs, ph);
        big_gemm<T, TU, TN, true, false, TM, UT, MM>(m, n, n, PB, ldpb, A, n, S, n, W + m, ldw, rank, CS, tiles, tcs, ph);
        ric_gemv<T, true>(m, n, Bm, m, g, r, 1, W + m + n, ldw, gw, nwc);  // column m+n of W
        ric_sync(CS);
        // phase 3: Cholesky of G (every CTA, own shared memory), [K | k] = -G^-1 [H | h]
        copy_rows_to_factor<T>(m, W, ldw, Ls, ldl);
        __syncthreads();
        if (!cta_chol<T>(m, Ls, ldl, dinv)) fail = min(fail, i + 1);
        for (int c0 = 2 * gw; c0 <= n; c0 += 2 * nwc) {
            const int c1 = c0 + 1 <= n ? c0 + 1 : c0;
            T b0[8], b1[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const int j = s * 32 + lane;
                b0[s] = j < m ? ldg_cg(W + (size_t)j * ldw + m + c0) : T(0);
                b1[s] = j < m ? ldg_cg(W + (size_t)j * ldw + m + c1) : T(0);
            }
            warp_chol_solve2_any<T>(m, Ls, ldl, dinv, b0, b1);
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const int j = s * 32 + lane;
                if (j >= m) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = h ? c1 : c0;
                    const T v = -(h ? b1[s] : b0[s]);
                    if (cc < n) {
                        Kw[(size_t)j * LD + cc] = v;
                        if (out.K) out.K[st * m * n + (size_t)j * n + cc] = v;
                    } else {
                        kw[j] = v;
                        if (out.k) out.k[st * m + j] = v;
                    }
                }
            }
        }
        ric_sync(CS);
        // phase 4: Abar = A + B K ; bbar = c + B k
        big_gemm<T, TN, TN, false, false, TM, UT, MM>(n, n, m, Bm, m, Kw, LD, A, n, Ab, LD, rank, CS, tiles, tcs, ph);
        ric_gemv<T, false>(n, m, Bm, m, kw, c, 1, bb, 1, gw, nwc);
        ric_sync(CS);
        // phase 5: V = P' Abar ; w = p' + P' bbar
        big_gemm<T, TN, TN, false, false, TM, UT, MM>(n, n, n, Pn, LD, Ab, LD, nullptr, 0, V, LD, rank, CS, tiles, tcs, ph);
        ric_gemv<T, false>(n, n, Pn, LD, bb, pn, 1, w, 1, gw, nwc);
        ric_sync(CS);
        // phase 6: P_i = Q + A^T V (+ S^T K) ; p_i = q + A^T w (+ S^T k)   (same tiles / rows: no barrier)
        big_gemm<T, TN, TN, true, false, TM, UT, MM>(n, n, n, A, n, V, LD, qp.Q + st * n * n, n, Pc, LD, rank, CS, tiles, tcs, ph);
        if (S) big_gemm<T, TN, TN, true, false, TM, UT, MM>(n, n, m, S, n, Kw, LD, Pc, LD, Pc, LD, rank, CS, tiles, tcs, ph);
        ric_gemv<T, true>(n, n, A, n, w, q, 1, pc, 1, gw, nwc);
        if (S) ric_gemv<T, true>(n, m, S, n, kw, pc, 1, pc, 1, gw, nwc);
        ric_sync(CS);
        // phase 7: re-symmetrise P_i (R22): upper-triangle pairs (r, c), (c, r) owned by one thread,
        // four pairs per batch with all loads issued before the stores
        {
            const int np = n * (n - 1) / 2, stride = CS * RIC_THREADS;
            for (int t0 = rank * RIC_THREADS + threadIdx.x; t0 < np; t0 += 4 * stride) {
                int ra[4], ca[4];
                T u[4], l[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    int t = t0 + e * stride;
                    ra[e] = -1;
                    if (t < np) {  // pair t -> (r, c), c > r: rows of the strict upper triangle
                        int rr = (int)((2 * n - 1 - sqrtf((float)((2 * n - 1) * (2 * n - 1) - 8 * t))) * 0.5f);
                        rr = max(0, min(rr, n - 2));
                        while (rr > 0 && rr * (2 * n - rr - 1) / 2 > t) --rr;
                        while ((rr + 1) * (2 * n - rr - 2) / 2 <= t) ++rr;
                        ra[e] = rr;
                        ca[e] = rr + 1 + (t - rr * (2 * n - rr - 1) / 2);
                        u[e] = ldg_cg(Pc + (size_t)ra[e] * LD + ca[e]);
                        l[e] = ldg_cg(Pc + (size_t)ca[e] * LD + ra[e]);
                    }
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (ra[e] >= 0) {
                        const T v = T(0.5) * (u[e] + l[e]);
                        Pc[(size_t)ra[e] * LD + ca[e]] = v;
                        Pc[(size_t)ca[e] * LD + ra[e]] = v;
                    }
                }
            }
        }
        ric_sync(CS);
    }
    (void)LDU;
    if constexpr (UT) tc_free(*tcs, RIC_TMEM_COLS);
    if (fail != INT_MAX && rank == 0 && threadIdx.x == 0) atomicMin(ws.fail + b, (2 << 24) | fail);
}

// Rows r0 .. r0+7 of y = op(x) for a row-major matrix A (ld lda) and a vector x in shared memory:
// one warp, lanes over k, all (row, k) loads of the 8 rows issued before the reduction (the forward
// recursion is one dependent gemv per stage, so memory-level parallelism is what sets its latency).
template <typename T>
__device__ __forceinline__ void warp_gemv8(int Mr, int K, const T *A, int lda, const T *x, int r0, T (&s)[8]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = T(0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // K <= 256
        const int k = lane + 32 * j;
        if (j * 32 < K) {
            const T xk = k < K ? x[k] : T(0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (r0 + q < Mr && k < K) s[q] = fma(ldg_cg(A + (size_t)(r0 + q) * lda + k), xk, s[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], off);
}

// Forward rollout of the large path, recursion only: dx_{i+1} = Abar_i dx_i + bbar_i (Eq. 15 with one
// chunk), one CTA per instance, dx_i kept in shared memory; du and dlam follow in k_big_tail.
template <typename T>
__global__ void __launch_bounds__(256) k_big_roll(const T *dx0, int B, int N, BigDims<T> d, BigWork<T> ws, T *dx_out) {
    __shared__ T xs[2][256];
    const int b = blockIdx.x;
    if (b >= B) return;
    const int n = d.n, LD = d.LD, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T *X = ws.dxw + (size_t)b * (N + 2) * LD;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const T v = dx0[(size_t)b * n + t];
        xs[0][t] = v;
        X[t] = v;
        dx_out[(size_t)b * (N + 2) * n + t] = v;
    }
    __syncthreads();
    for (int i = 0; i <= N; ++i) {
        const T *Te = ws.tel + ((size_t)b * (N + 1) + i) * d.psize(), *tb = Te + (size_t)n * LD;
        const T *xc = xs[i & 1];
        T *xn = xs[(i + 1) & 1];
        for (int r0 = 8 * wid; r0 < n; r0 += 8 * (blockDim.x >> 5)) {
            T s[8];
            warp_gemv8<T>(n, n, Te, LD, xc, r0, s);
            if (lane < 8 && r0 + lane < n) {
                const int r = r0 + lane;
                T v = s[0];
#pragma unroll
                for (int q = 1; q < 8; ++q) v = lane == q ? s[q] : v;
                v += ldg_cg(tb + r);
                xn[r] = v;
                X[(size_t)(i + 1) * LD + r] = v;
                dx_out[((size_t)b * (N + 2) + i + 1) * n + r] = v;
            }
        }
        __syncthreads();
    }
}

// du_i = K_i dx_i + k_i (Eq. 6, i <= N) and dlam_i = P_i dx_i + p_i (Eq. 7, i <= N+1), after the
// recursion.  HBM-bound: it streams every P_i and K_i once (algorithmic bytes (n + m) LD per stage).
// One block of 128 threads per (instance, stage) item, dx_i staged in shared memory, one thread per
// output row: the row is read with independent 16-byte L2-only loads (rows are 16-byte aligned, LD a
// multiple of 4), so every thread keeps ceil(n / 4) loads in flight and every fetched sector is used.
template <typename T>
__global__ void __launch_bounds__(128) k_big_tail(int B, int N, BigDims<T> d, BigWork<T> ws, LqOut<T> out) {
    __shared__ __align__(16) T xs[256];
    const int n = d.n, m = d.m, LD = d.LD;
    const long item = blockIdx.x;
    const int b = (int)(item / (N + 2)), i = (int)(item % (N + 2));
    if (b >= B) return;
    for (int t = threadIdx.x; t < LD; t += blockDim.x)
        xs[t] = t < n ? ldg_cg(ws.dxw + ((size_t)b * (N + 2) + i) * LD + t) : T(0);
    __syncthreads();
    const T *Pi = ws.Pp + ((size_t)b * (N + 2) + i) * d.psize();
    const size_t st = (size_t)b * (N + 1) + (i <= N ? i : 0);
    const T *Kw = ws.Kk + st * d.ksize();
    const int rows = n + (i <= N ? m : 0);
    constexpr int V = 16 / (int)sizeof(T);
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const bool isP = r < n;
        const T *row = isP ? Pi + (size_t)r * LD : Kw + (size_t)(r - n) * LD;
        T acc0 = T(0), acc1 = T(0);
        int k = 0;
        for (; k + 2 * V <= LD; k += 2 * V) {
            if constexpr (sizeof(T) == 4) {
                const float4 a = __ldcg(reinterpret_cast<const float4 *>(row + k));
                const float4 c = __ldcg(reinterpret_cast<const float4 *>(row + k + 4));
                acc0 = fma(a.x, xs[k], acc0); acc1 = fma(a.y, xs[k + 1], acc1);
                acc0 = fma(a.z, xs[k + 2], acc0); acc1 = fma(a.w, xs[k + 3], acc1);
                acc0 = fma(c.x, xs[k + 4], acc0); acc1 = fma(c.y, xs[k + 5], acc1);
                acc0 = fma(c.z, xs[k + 6], acc0); acc1 = fma(c.w, xs[k + 7], acc1);
            } else {
                const double2 a = __ldcg(reinterpret_cast<const double2 *>(row + k));
                const double2 c = __ldcg(reinterpret_cast<const double2 *>(row + k + 2));
                acc0 = fma(a.x, xs[k], acc0); acc1 = fma(a.y, xs[k + 1], acc1);
                acc0 = fma(c.x, xs[k + 2], acc0); acc1 = fma(c.y, xs[k + 3], acc1);
            }
        }
        for (; k < LD; ++k) acc0 = fma(ldg_cg(row + k), xs[k], acc0);   // padding columns hold zeros in xs
        const T v = acc0 + acc1;
        if (isP) out.dlam[((size_t)b * (N + 2) + i) * n + r] = v + Pi[(size_t)n * LD + r];
        else out.du[st * m + (r - n)] = v + Kw[(size_t)m * LD + (r - n)];
    }
}

// R_i SPD check of Eq. 12 for every (instance, stage), persistent CTAs; a failure at stage
// i is reported as i + 1 with the element-initialisation rank (ahead of the policy's G failures).
template <typename T>
__global__ void __launch_bounds__(256) k_big_rchk(const T *R, int B, int N, int m, int32_t *fail) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const int ldl = ric_ldl(m);
    T *Ls = reinterpret_cast<T *>(dyn), *dinv = Ls + (size_t)m * ldl;
    for (long item = blockIdx.x; item < (long)B * (N + 1); item += gridDim.x) {
        const int b = (int)(item / (N + 1)), i = (int)(item % (N + 1));
        const T *Ri = R + (size_t)item * m * m;
        copy_rows_to_factor<T>(m, Ri, m, Ls, ldl);
        __syncthreads();
        const bool ok = cta_chol<T>(m, Ls, ldl, dinv);
        if (!ok && threadIdx.x == 0) atomicMin(fail + b, i + 1);
        __syncthreads();
    }
}

}  // namespace pdilqr
