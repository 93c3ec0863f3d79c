// big.cuh -- large-dimension path (16 < max(n, m) <= 256: configs 4 and 5) of the
// same LQ/KKT solve, single-chunk schedule (s_i = e_i (x) s_{i+1}, cheap rule), CTA-level dense
// algebra on matrices kept in global memory (L2-resident per instance) and staged through shared
// memory tiles:
//   cta_gemm      C = alpha op(A) op(B) + beta C, 64x64 output tiles, 16-deep k panels, 4x4
//                 register micro-tiles per thread (256 threads)
//   cta_gj        Gauss-Jordan with partial pivoting (explicit row swaps) on W = [M | RHS]
// Kernels (one launch each):
//   k_big_init    Eq. 12/13 elements, persistent CTAs over (instance, stage)
//   k_big_fold    reverse scan, one CTA per instance (Eq. 11 cheap rule, R1-R2, R22)
//   k_big_policy  Eq. 5 rows + Eq. 14, persistent CTAs over (instance, stage)
//   k_big_fwd     Eq. 15 rollout with one chunk, du (Eq. 6), dlam (Eq. 7), one CTA per instance
// Matrices are row-major with the padded leading dimension LD = round_up(n, 4) (LDU for m).
#pragma once

#include "lq.cuh"

namespace pdilqr {

constexpr int BIG_THREADS = 256;

__host__ __device__ constexpr int ld_of(int d) { return (d + 3) & ~3; }

template <typename T>
struct GemmSmem {
    T As[16][64 + 4];
    T Bs[16][64 + 4];
};

// C[Mr x Nc] = alpha * op(A)[Mr x K] * op(B)[K x Nc] + beta * C.  op(A) = A (row-major Mr x K,
// leading dim lda) or A^T (A stored K x Mr); same for B.  C must not alias A or B.  All threads of
// the CTA must call it; ends with __syncthreads.
template <typename T, bool TA, bool TB>
__device__ void cta_gemm(int Mr, int Nc, int K, T alpha, const T *A, int lda, const T *Bm, int ldb, T beta, T *C,
                         int ldc, GemmSmem<T> &sm) {
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    for (int tm = 0; tm < Mr; tm += 64) {
        for (int tn = 0; tn < Nc; tn += 64) {
            T acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] = T(0);
            // k panels of 16, the next panel is loaded into registers while the current one is used
            T pa[4], pb[4];
            auto fetch = [&](int k0) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int idx = tid + e * BIG_THREADS;  // 0..1023
                    const int kk = idx >> 6, mm = idx & 63;  // As[kk][mm] = opA(tm+mm, k0+kk)
                    const int r = tm + mm, c = k0 + kk;
                    pa[e] = (r < Mr && c < K) ? (TA ? A[(size_t)c * lda + r] : A[(size_t)r * lda + c]) : T(0);
                    const int rb = k0 + kk, cb = tn + mm;  // Bs[kk][nn] = opB(k0+kk, tn+nn)
                    pb[e] = (rb < K && cb < Nc) ? (TB ? Bm[(size_t)cb * ldb + rb] : Bm[(size_t)rb * ldb + cb]) : T(0);
                }
            };
            fetch(0);
            for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int idx = tid + e * BIG_THREADS;
                    sm.As[idx >> 6][idx & 63] = pa[e];
                    sm.Bs[idx >> 6][idx & 63] = pb[e];
                }
                __syncthreads();
                if (k0 + 16 < K) fetch(k0 + 16);
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) {
                    T a[4], b[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) { a[q] = sm.As[kk][ty * 4 + q]; b[q] = sm.Bs[kk][tx * 4 + q]; }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int w = 0; w < 4; ++w) acc[q][w] = fma(a[q], b[w], acc[q][w]);
                }
                __syncthreads();
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = tm + ty * 4 + q;
                if (r >= Mr) continue;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const int c = tn + tx * 4 + w;
                    if (c < Nc) {
                        T *p = C + (size_t)r * ldc + c;
                        *p = beta == T(0) ? alpha * acc[q][w] : fma(alpha, acc[q][w], beta * *p);
                    }
                }
            }
        }
    }
    __syncthreads();
}

// y[r] = beta*y[r] + alpha * sum_k op(A)[r][k] x[k], r < Mr (CTA-cooperative, one warp per row).
template <typename T, bool TA>
__device__ void cta_gemv(int Mr, int K, T alpha, const T *A, int lda, const T *x, T beta, T *y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = BIG_THREADS / 32;
    for (int r = wid; r < Mr; r += nw) {
        T s = T(0);
        for (int k = lane; k < K; k += 32) s = fma(TA ? A[(size_t)k * lda + r] : A[(size_t)r * lda + k], x[k], s);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) y[r] = beta == T(0) ? alpha * s : fma(alpha, s, beta * y[r]);
    }
    __syncthreads();
}

struct GjShared {
    float rv[BIG_THREADS / 32];
    int ri[BIG_THREADS / 32];
    int piv;
    int ok;
};

// Solve M X = RHS with W = [M | RHS] (n rows, n + nrhs columns, row-major, leading dim ldw),
// Gauss-Jordan with partial pivoting and explicit row swaps; on return W[:, n:] = X (rows in the
// original order).  PIVOT = false for SPD M (pivots must stay > 0).  Returns false if a pivot is
// zero / non-finite (or <= 0 without pivoting).
template <typename T, bool PIVOT>
__device__ bool cta_gj(int n, int nrhs, T *W, int ldw, GjShared &gs) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = BIG_THREADS / 32;
    const int ncol = n + nrhs;
    if (tid == 0) gs.ok = 1;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        int p = k;
        if constexpr (PIVOT) {
            float bv = -1.f;
            int bi = k;
            for (int i = k + tid; i < n; i += BIG_THREADS) {
                const float v = fabsf((float)W[(size_t)i * ldw + k]);
                if (v > bv || (v == bv && i < bi) || !(v == v)) { bv = (v == v) ? v : INFINITY; bi = i; }
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) { gs.rv[wid] = bv; gs.ri[wid] = bi; }
            __syncthreads();
            if (tid == 0) {
                float b2 = gs.rv[0];
                int i2 = gs.ri[0];
                for (int w = 1; w < nw; ++w)
                    if (gs.rv[w] > b2 || (gs.rv[w] == b2 && gs.ri[w] < i2)) { b2 = gs.rv[w]; i2 = gs.ri[w]; }
                gs.piv = i2;
            }
            __syncthreads();
            p = gs.piv;
            if (p != k)
                for (int j = tid; j < ncol; j += BIG_THREADS) {
                    const T t = W[(size_t)k * ldw + j];
                    W[(size_t)k * ldw + j] = W[(size_t)p * ldw + j];
                    W[(size_t)p * ldw + j] = t;
                }
            __syncthreads();
        }
        const T pv = W[(size_t)k * ldw + k];
        const bool good = PIVOT ? (pv != T(0) && isfinite(pv)) : (pv > T(0) && isfinite(pv));
        if (!good && tid == 0) gs.ok = 0;
        const T inv = T(1) / pv;
        // normalise the pivot row (columns > k), then eliminate column k from every other row
        for (int j = k + 1 + tid; j < ncol; j += BIG_THREADS) W[(size_t)k * ldw + j] *= inv;
        __syncthreads();
        const int width = ncol - k - 1;
        for (int i = wid; i < n; i += nw) {
            if (i == k) continue;
            const T f = W[(size_t)i * ldw + k];
            if (f == T(0)) continue;
            T *wi = W + (size_t)i * ldw;
            const T *wk = W + (size_t)k * ldw;
            for (int j = k + 1 + lane; j < k + 1 + width; j += 32) wi[j] = fma(-f, wk[j], wi[j]);
        }
        __syncthreads();
    }
    const bool ok = gs.ok != 0;
    __syncthreads();
    return ok;
}

template <typename T>
__device__ void cta_symmetrize(int n, T *P, int ld) {
    for (int t = threadIdx.x; t < n * n; t += BIG_THREADS) {
        const int r = t / n, c = t % n;
        if (c > r) {
            const T v = T(0.5) * (P[(size_t)r * ld + c] + P[(size_t)c * ld + r]);
            P[(size_t)r * ld + c] = v;
            P[(size_t)c * ld + r] = v;
        }
    }
    __syncthreads();
}

// Workspace views of the large path (element layout: A, C, P with leading dim LD, then b, p).
template <typename T>
struct BigWork {
    T *elems;    // [B][N+2][3 n LD + 2 LD]
    T *Pp;       // [B][N+2][n LD + LD]
    T *Kk;       // [B][N+1][m LD + LDU]    K (m x n, ld LD), k
    T *tel;      // [B][N+1][n LD + LD]     Abar, bbar
    T *dxw;      // [B][N+2][LD]
    T *scratch;  // per-CTA slots of `slot` values
    size_t slot;
    int32_t *fail;
};

template <typename T>
struct BigDims {
    int n, m, LD, LDU;
    __device__ size_t esize() const { return (size_t)3 * n * LD + 2 * LD; }
    __device__ size_t psize() const { return (size_t)n * LD + LD; }
    __device__ size_t ksize() const { return (size_t)m * LD + LDU; }
};

// -------------------------------------------------------------------------- element init
// Per stage i <= N: W = [R | S | r | B^T] (m rows, ld = m + 2n + 1 padded), GJ without pivoting
// (R SPD), then A~ = A - B Z_S, C~ = B Z_B, P~ = Q - S^T Z_S, b~ = b - B z_r, p~ = q - S^T z_r.
// Terminal (i = N+1): A~ = C~ = b~ = 0, P~ = P_{N+1}, p~ = p_{N+1}.
template <typename T>
__global__ void __launch_bounds__(BIG_THREADS) k_big_init(LqArgs<T> qp, int B, int N, BigDims<T> d, BigWork<T> ws,
                                                          int w_in_smem) {
    __shared__ GemmSmem<T> gsm;
    __shared__ GjShared gjs;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = d.n, m = d.m, LD = d.LD;
    const int ldw = ld_of(m + 2 * n + 1);
    T *W = w_in_smem ? reinterpret_cast<T *>(dyn) : ws.scratch + (size_t)blockIdx.x * ws.slot;
    for (long item = blockIdx.x; item < (long)B * (N + 2); item += gridDim.x) {
        const int b = (int)(item / (N + 2)), i = (int)(item % (N + 2));
        T *e = ws.elems + ((size_t)b * (N + 2) + i) * d.esize();
        T *eA = e, *eC = e + (size_t)n * LD, *eP = e + (size_t)2 * n * LD, *eb = e + (size_t)3 * n * LD, *ep = eb + LD;
        if (i == N + 1) {
            for (int t = threadIdx.x; t < n * n; t += BIG_THREADS) {
                const int r = t / n, c = t % n;
                eA[(size_t)r * LD + c] = T(0);
                eC[(size_t)r * LD + c] = T(0);
                eP[(size_t)r * LD + c] = qp.Pt[(size_t)b * n * n + t];
            }
            for (int r = threadIdx.x; r < n; r += BIG_THREADS) { eb[r] = T(0); ep[r] = qp.pt[(size_t)b * n + r]; }
            __syncthreads();
            continue;
        }
        const size_t st = (size_t)b * (N + 1) + i;
        const T *A = qp.A + st * n * n, *Bm = qp.Bm + st * n * m, *R = qp.R + st * m * m;
        const T *S = qp.S ? qp.S + st * m * n : nullptr, *q = qp.q + st * n, *r = qp.r + st * m, *c = qp.c + st * n;
        for (int t = threadIdx.x; t < m * (m + 2 * n + 1); t += BIG_THREADS) {
            const int row = t / (m + 2 * n + 1), col = t % (m + 2 * n + 1);
            T v;
            if (col < m) v = R[(size_t)row * m + col];
            else if (col < m + n) v = S ? S[(size_t)row * n + (col - m)] : T(0);
            else if (col == m + n) v = r[row];
            else v = Bm[(size_t)(col - m - n - 1) * m + row];  // B^T
            W[(size_t)row * ldw + col] = v;
        }
        __syncthreads();
        if (!cta_gj<T, false>(m, 2 * n + 1, W, ldw, gjs) && threadIdx.x == 0) atomicMin(ws.fail + b, i + 1);
        const T *ZS = W + m, *zr = W + m + n, *ZB = W + m + n + 1;   // rows of R^-1 [S | r | B^T]
        // A~ = A - B Z_S ;  C~ = B Z_B ;  P~ = Q - S^T Z_S
        for (int t = threadIdx.x; t < n * n; t += BIG_THREADS) {
            const int rr = t / n, cc = t % n;
            eA[(size_t)rr * LD + cc] = A[t];
            eP[(size_t)rr * LD + cc] = qp.Q[st * n * n + t];
        }
        __syncthreads();
        cta_gemm<T, false, false>(n, n, m, T(-1), Bm, m, ZS, ldw, T(1), eA, LD, gsm);
        cta_gemm<T, false, false>(n, n, m, T(1), Bm, m, ZB, ldw, T(0), eC, LD, gsm);
        if (S) cta_gemm<T, true, false>(n, n, m, T(-1), S, n, ZS, ldw, T(1), eP, LD, gsm);
        {   // b~ = b - B z_r ;  p~ = q - S^T z_r   (z_r = column m+n of W), one warp per row
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            for (int rr = wid; rr < n; rr += BIG_THREADS / 32) {
                T sb = T(0), sp = T(0);
                for (int k = lane; k < m; k += 32) {
                    const T z = W[(size_t)k * ldw + m + n];
                    sb = fma(Bm[(size_t)rr * m + k], z, sb);
                    if (S) sp = fma(S[(size_t)k * n + rr], z, sp);
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    sb += __shfl_xor_sync(0xffffffffu, sb, off);
                    sp += __shfl_xor_sync(0xffffffffu, sp, off);
                }
                if (lane == 0) { eb[rr] = c[rr] - sb; ep[rr] = q[rr] - sp; }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------- reverse scan (fold)
// One CTA per instance: s_{N+1} = e_{N+1}; for i = N..0:  M = I + C~_i P', W = [M | A~_i],
// X = M^-1 A~_i (pivoted GJ), w = p' + P' b~_i, V = P' X, P_i = A~_i^T V + P~_i (symmetrised),
// p_i = X^T w + p~_i.  Scratch slot: P' (n LD), W (n x ld(2n)), V (n LD), w, p' (LD each).
template <typename T>
__global__ void __launch_bounds__(BIG_THREADS) k_big_fold(int B, int N, BigDims<T> d, BigWork<T> ws, int w_in_smem) {
    __shared__ GemmSmem<T> gsm;
    __shared__ GjShared gjs;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int b = blockIdx.x;
    if (b >= B) return;
    const int n = d.n, LD = d.LD, ldw = ld_of(2 * n);
    T *Pc = ws.scratch + (size_t)blockIdx.x * ws.slot;
    T *Wg = Pc + (size_t)n * LD, *V = Wg + (size_t)n * ldw, *w = V + (size_t)n * LD, *pc = w + LD;
    T *W = w_in_smem ? reinterpret_cast<T *>(dyn) : Wg;
    const T *E = ws.elems + (size_t)b * (N + 2) * d.esize();
    T *Pp = ws.Pp + (size_t)b * (N + 2) * d.psize();
    {   // s_{N+1}
        const T *e = E + (size_t)(N + 1) * d.esize();
        for (int t = threadIdx.x; t < n * LD; t += BIG_THREADS) {
            Pc[t] = e[(size_t)2 * n * LD + t];
            Pp[(size_t)(N + 1) * d.psize() + t] = Pc[t];
        }
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) {
            pc[t] = e[(size_t)3 * n * LD + LD + t];
            Pp[(size_t)(N + 1) * d.psize() + (size_t)n * LD + t] = pc[t];
        }
        __syncthreads();
    }
    int fail = INT_MAX;
    for (int i = N; i >= 0; --i) {
        const T *e = E + (size_t)i * d.esize();
        const T *eA = e, *eC = e + (size_t)n * LD, *eP = e + (size_t)2 * n * LD, *eb = e + (size_t)3 * n * LD,
                *ep = eb + LD;
        // W[:, :n] = I + C~ P' ; W[:, n:] = A~
        for (int t = threadIdx.x; t < n * n; t += BIG_THREADS) {
            const int r = t / n, c = t % n;
            W[(size_t)r * ldw + c] = (r == c) ? T(1) : T(0);
            W[(size_t)r * ldw + n + c] = eA[(size_t)r * LD + c];
        }
        __syncthreads();
        cta_gemm<T, false, false>(n, n, n, T(1), eC, LD, Pc, LD, T(1), W, ldw, gsm);
        cta_gemv<T, false>(n, n, T(1), Pc, LD, eb, T(0), w);       // P' b~
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) w[t] += pc[t];  // w = p' + P' b~
        __syncthreads();
        if (!cta_gj<T, true>(n, n, W, ldw, gjs)) fail = min(fail, i + 1);
        const T *X = W + n;                                          // ld = ldw
        cta_gemm<T, false, false>(n, n, n, T(1), Pc, LD, X, ldw, T(0), V, LD, gsm);   // V = P' X
        // p_i = X^T w + p~  (into pc after reading w), P_i = A~^T V + P~ (into Pc)
        cta_gemv<T, true>(n, n, T(1), X, ldw, w, T(0), pc);
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) pc[t] += ep[t];
        for (int t = threadIdx.x; t < n * LD; t += BIG_THREADS) Pc[t] = eP[t];
        __syncthreads();
        cta_gemm<T, true, false>(n, n, n, T(1), eA, LD, V, LD, T(1), Pc, LD, gsm);
        cta_symmetrize<T>(n, Pc, LD);
        T *Po = Pp + (size_t)i * d.psize();
        for (int t = threadIdx.x; t < n * LD; t += BIG_THREADS) Po[t] = Pc[t];
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) Po[(size_t)n * LD + t] = pc[t];
        __syncthreads();
    }
    if (fail != INT_MAX && threadIdx.x == 0) atomicMin(ws.fail + b, (1 << 24) | fail);
}

// ------------------------------------------------- reverse associative scan for large n (tree)
// One Kogge-Stone level of the reverse scan over the N+2 value elements (Eq. 11 full rule
// with readings R1-R3; the small-n path's D9 order): for every instance b and j < L - dl,
// dst_j = src_j (x) src_{j+dl}; the elements with j + dl >= L are already complete suffixes and are
// copied.  One CTA per combine (persistent over (instance, j)), CTA-level dense algebra with the
// pivoted Gauss-Jordan on W = [I + C1 P2 | A1 | C1 | b1 - C1 p2]:
//   X = M^-1 A1, Y = M^-1 C1, z = M^-1 (b1 - C1 p2);  A = A2 X,  b = A2 z + b2,
//   C = A2 Y A2^T + C2,  P = A1^T (P2 X) + P1,  p = X^T (p2 + P2 b1) + p1   (C, P re-symmetrised, R22).
// Scratch slot: W (n x ld(3n+1), global unless it fits shared memory), T1 (n x LD), two vectors.
template <typename T>
__global__ void __launch_bounds__(BIG_THREADS) k_bigks_level(int B, int N, int dl, BigDims<T> d, BigWork<T> ws,
                                                             const T *src, T *dst, int w_in_smem) {
    __shared__ GemmSmem<T> gsm;
    __shared__ GjShared gjs;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = d.n, LD = d.LD, ldw = ld_of(3 * n + 1), L = N + 2;
    const size_t es = d.esize();
    T *slot = ws.scratch + (size_t)blockIdx.x * ws.slot;
    T *W = w_in_smem ? reinterpret_cast<T *>(dyn) : slot;
    T *T1 = slot + (size_t)n * ldw, *v1 = T1 + (size_t)n * LD, *v2 = v1 + LD;
    for (long item = blockIdx.x; item < (long)B * L; item += gridDim.x) {
        const int b = (int)(item / L), j = (int)(item % L);
        const T *e1 = src + ((size_t)b * L + j) * es;
        T *o = dst + ((size_t)b * L + j) * es;
        if (j + dl >= L) {   // complete suffix: unchanged
            for (size_t t = threadIdx.x; t < es; t += BIG_THREADS) o[t] = e1[t];
            __syncthreads();
            continue;
        }
        const T *e2 = src + ((size_t)b * L + j + dl) * es;
        const T *A1 = e1, *C1 = e1 + (size_t)n * LD, *P1 = e1 + (size_t)2 * n * LD, *b1 = e1 + (size_t)3 * n * LD, *p1 = b1 + LD;
        const T *A2 = e2, *C2 = e2 + (size_t)n * LD, *P2 = e2 + (size_t)2 * n * LD, *b2 = e2 + (size_t)3 * n * LD, *p2 = b2 + LD;
        T *oA = o, *oC = o + (size_t)n * LD, *oP = o + (size_t)2 * n * LD, *ob = o + (size_t)3 * n * LD, *op = ob + LD;
        cta_gemv<T, false>(n, n, T(1), C1, LD, p2, T(0), v1);            // C1 p2
        for (int t = threadIdx.x; t < n * (3 * n + 1); t += BIG_THREADS) {
            const int r = t / (3 * n + 1), c = t - r * (3 * n + 1);
            T v;
            if (c < n) v = (r == c) ? T(1) : T(0);
            else if (c < 2 * n) v = A1[(size_t)r * LD + (c - n)];
            else if (c < 3 * n) v = C1[(size_t)r * LD + (c - 2 * n)];
            else v = b1[r] - v1[r];
            W[(size_t)r * ldw + c] = v;
        }
        __syncthreads();
        cta_gemm<T, false, false>(n, n, n, T(1), C1, LD, P2, LD, T(1), W, ldw, gsm);   // M = I + C1 P2
        if (!cta_gj<T, true>(n, 2 * n + 1, W, ldw, gjs) && threadIdx.x == 0) atomicMin(ws.fail + b, (1 << 24) | (j + 1));
        const T *X = W + n, *Y = W + 2 * n;
        for (int r = threadIdx.x; r < n; r += BIG_THREADS) v2[r] = W[(size_t)r * ldw + 3 * n];   // z
        __syncthreads();
        cta_gemm<T, false, false>(n, n, n, T(1), A2, LD, X, ldw, T(0), oA, LD, gsm);           // A = A2 X
        cta_gemv<T, false>(n, n, T(1), A2, LD, v2, T(0), ob);                                  // A2 z
        for (int r = threadIdx.x; r < n; r += BIG_THREADS) ob[r] += b2[r];
        __syncthreads();
        cta_gemm<T, false, true>(n, n, n, T(1), Y, ldw, A2, LD, T(0), T1, LD, gsm);            // Y A2^T
        for (int t = threadIdx.x; t < n * LD; t += BIG_THREADS) oC[t] = C2[t];
        __syncthreads();
        cta_gemm<T, false, false>(n, n, n, T(1), A2, LD, T1, LD, T(1), oC, LD, gsm);          // C = A2 Y A2^T + C2
        cta_gemm<T, false, false>(n, n, n, T(1), P2, LD, X, ldw, T(0), T1, LD, gsm);           // P2 X
        for (int t = threadIdx.x; t < n * LD; t += BIG_THREADS) oP[t] = P1[t];
        __syncthreads();
        cta_gemm<T, true, false>(n, n, n, T(1), A1, LD, T1, LD, T(1), oP, LD, gsm);           // P = A1^T P2 X + P1
        cta_gemv<T, false>(n, n, T(1), P2, LD, b1, T(0), v1);                                  // P2 b1
        for (int r = threadIdx.x; r < n; r += BIG_THREADS) v1[r] += p2[r];                    // w
        __syncthreads();
        cta_gemv<T, true>(n, n, T(1), X, ldw, v1, T(0), op);                                   // X^T w
        for (int r = threadIdx.x; r < n; r += BIG_THREADS) op[r] += p1[r];
        __syncthreads();
        cta_symmetrize<T>(n, oC, LD);
        cta_symmetrize<T>(n, oP, LD);
    }
}

// Read-out after the last level: (P_i, p_i) = (P~, p~) of the complete suffix s_i (reading R5).
template <typename T>
__global__ void k_bigks_readout(int B, int N, BigDims<T> d, const T *s, T *Pp) {
    const int L = N + 2, n = d.n, LD = d.LD;
    const size_t es = d.esize(), ps = d.psize();
    const long tot = (long)B * L * (long)ps;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long)gridDim.x * blockDim.x) {
        const long el = t / (long)ps;
        const size_t k = (size_t)(t - el * (long)ps);
        const T *e = s + (size_t)el * es;
        Pp[(size_t)el * ps + k] = k < (size_t)n * LD ? e[(size_t)2 * n * LD + k] : e[(size_t)3 * n * LD + LD + (k - (size_t)n * LD)];
    }
}

// ------------------------------------------------------------------------------- policy
// Per stage: PB = P_{i+1} B, g = p_{i+1} + P_{i+1} b; W = [G | H | h] with G = R + B^T PB,
// H = S + PB^T A, h = B^T g + r; GJ (SPD) -> K = -G^-1 H, k = -G^-1 h; Abar = A + B K,
// bbar = B k + b.  Scratch: PB (n x ld(m)), W (m x ld(m+n+1)), g (LD).
template <typename T>
__global__ void __launch_bounds__(BIG_THREADS) k_big_policy(LqArgs<T> qp, int B, int N, BigDims<T> d, BigWork<T> ws,
                                                            LqOut<T> out, int w_in_smem) {
    __shared__ GemmSmem<T> gsm;
    __shared__ GjShared gjs;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = d.n, m = d.m, LD = d.LD, ldpb = ld_of(m), ldw = ld_of(m + n + 1);
    T *PB = ws.scratch + (size_t)blockIdx.x * ws.slot;
    T *Wg = PB + (size_t)n * ldpb, *g = Wg + (size_t)m * ldw;
    T *W = w_in_smem ? reinterpret_cast<T *>(dyn) : Wg;
    for (long item = blockIdx.x; item < (long)B * (N + 1); item += gridDim.x) {
        const int b = (int)(item / (N + 1)), i = (int)(item % (N + 1));
        const size_t st = (size_t)b * (N + 1) + i;
        const T *A = qp.A + st * n * n, *Bm = qp.Bm + st * n * m, *R = qp.R + st * m * m;
        const T *S = qp.S ? qp.S + st * m * n : nullptr, *r = qp.r + st * m, *c = qp.c + st * n;
        const T *Pn = ws.Pp + ((size_t)b * (N + 2) + i + 1) * d.psize(), *pn = Pn + (size_t)n * LD;
        cta_gemm<T, false, false>(n, m, n, T(1), Pn, LD, Bm, m, T(0), PB, ldpb, gsm);   // PB = P' B
        cta_gemv<T, false>(n, n, T(1), Pn, LD, c, T(0), g);
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) g[t] += pn[t];
        for (int t = threadIdx.x; t < m * (m + n + 1); t += BIG_THREADS) {
            const int row = t / (m + n + 1), col = t % (m + n + 1);
            T v;
            if (col < m) v = R[(size_t)row * m + col];
            else if (col < m + n) v = S ? S[(size_t)row * n + (col - m)] : T(0);
            else v = r[row];
            W[(size_t)row * ldw + col] = v;
        }
        __syncthreads();
        cta_gemm<T, true, false>(m, m, n, T(1), Bm, m, PB, ldpb, T(1), W, ldw, gsm);       // G += B^T PB
        cta_gemm<T, true, false>(m, n, n, T(1), PB, ldpb, A, n, T(1), W + m, ldw, gsm);   // H += PB^T A
        {   // h += B^T g  (column m+n of W)
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            for (int rr = wid; rr < m; rr += BIG_THREADS / 32) {
                T sacc = T(0);
                for (int k = lane; k < n; k += 32) sacc = fma(Bm[(size_t)k * m + rr], g[k], sacc);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
                if (lane == 0) W[(size_t)rr * ldw + m + n] += sacc;
            }
        }
        __syncthreads();
        if (!cta_gj<T, false>(m, n + 1, W, ldw, gjs) && threadIdx.x == 0) atomicMin(ws.fail + b, (2 << 24) | (i + 1));
        // K = -sol, k = -sol (m rows); store policy, Abar = A + B K, bbar = B k + b
        T *Kw = ws.Kk + st * d.ksize(), *kw = Kw + (size_t)m * LD;
        for (int t = threadIdx.x; t < m * n; t += BIG_THREADS) {
            const int rr = t / n, cc = t % n;
            const T v = -W[(size_t)rr * ldw + m + cc];
            Kw[(size_t)rr * LD + cc] = v;
            if (out.K) out.K[st * m * n + t] = v;
        }
        for (int t = threadIdx.x; t < m; t += BIG_THREADS) {
            const T v = -W[(size_t)t * ldw + m + n];
            kw[t] = v;
            if (out.k) out.k[st * m + t] = v;
        }
        T *Te = ws.tel + st * d.psize(), *tb = Te + (size_t)n * LD;
        for (int t = threadIdx.x; t < n * n; t += BIG_THREADS) Te[(size_t)(t / n) * LD + t % n] = A[t];
        __syncthreads();
        cta_gemm<T, false, false>(n, n, m, T(1), Bm, m, Kw, LD, T(1), Te, LD, gsm);
        cta_gemv<T, false>(n, m, T(1), Bm, m, kw, T(0), tb);
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) tb[t] += c[t];
        __syncthreads();
    }
}

// ------------------------------------------------------- forward rollout, du, dlam (one CTA)
template <typename T>
__global__ void __launch_bounds__(BIG_THREADS) k_big_fwd(const T *dx0, int B, int N, BigDims<T> d, BigWork<T> ws,
                                                         LqOut<T> out) {
    const int b = blockIdx.x;
    if (b >= B) return;
    const int n = d.n, m = d.m, LD = d.LD;
    T *X = ws.dxw + (size_t)b * (N + 2) * LD;
    for (int t = threadIdx.x; t < n; t += BIG_THREADS) {
        X[t] = dx0[(size_t)b * n + t];
        out.dx[(size_t)b * (N + 2) * n + t] = X[t];
    }
    __syncthreads();
    for (int i = 0; i <= N; ++i) {
        const size_t st = (size_t)b * (N + 1) + i;
        const T *Te = ws.tel + st * d.psize(), *Kw = ws.Kk + st * d.ksize();
        cta_gemv<T, false>(n, n, T(1), Te, LD, X + (size_t)i * LD, T(0), X + (size_t)(i + 1) * LD);
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) {
            X[(size_t)(i + 1) * LD + t] += Te[(size_t)n * LD + t];
        }
        __syncthreads();
        T *du = out.du + st * m;
        cta_gemv<T, false>(m, n, T(1), Kw, LD, X + (size_t)i * LD, T(0), du);
        for (int t = threadIdx.x; t < m; t += BIG_THREADS) du[t] += Kw[(size_t)m * LD + t];
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) out.dx[((size_t)b * (N + 2) + i + 1) * n + t] = X[(size_t)(i + 1) * LD + t];
        __syncthreads();
    }
    for (int i = 0; i <= N + 1; ++i) {  // dlam_i = P_i dx_i + p_i
        const T *Pi = ws.Pp + ((size_t)b * (N + 2) + i) * d.psize();
        T *dl = out.dlam + ((size_t)b * (N + 2) + i) * n;
        cta_gemv<T, false>(n, n, T(1), Pi, LD, X + (size_t)i * LD, T(0), dl);
        for (int t = threadIdx.x; t < n; t += BIG_THREADS) dl[t] += Pi[(size_t)n * LD + t];
        __syncthreads();
    }
}

}  // namespace pdilqr
