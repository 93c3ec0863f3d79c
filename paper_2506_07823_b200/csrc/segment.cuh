// segment.cuh -- horizon sharding of one LQ problem over ranks (NEXT-2 of SURVEY §8(f); the
// associative scans of P:188-271 split at chunk boundaries).  Rank r holds the stages [s_r, e_r)
// of the global horizon as an ordinary LQ handle (its own N+1 stages; its terminal node is the
// global node e_r).  Because the combination rule is associative (Eq. 8), the global suffix at e_r is
//   T_r = S_{r+1} (x) ... (x) S_{G-1} (x) e_term,   S_j = e_{s_j} (x) ... (x) e_{e_j - 1}
// (chunk summaries by the full rule, Eq. 11 as corrected in R1/R2), a suffix whose (P, p) is the
// value function at e_r: the rank's local LQ with P_{N+1} := P(T_r), p_{N+1} := p(T_r) has exactly
// the global solution on its stages.  Forward, the closed-loop maps compose (Eq. 15, R6): the state
// at s_r is F_{r-1} o ... o F_0 (dx0), F_j = (Phi_j, phi_j) the chunk's affine map dx_s -> dx_e.
//   k_seg_reduce   S = e_0 (x) ... (x) e_N of every instance: in-place tree reduction of the
//                  element array (one CTA per instance, one worker per combine, log2 depth)
//   k_seg_suffix   (P, p) of S_{r+1} (x) ... (x) S_{G-1} (x) (P_term, p_term) (cheap rule, right to left)
//   k_seg_forward  (Phi, phi) = composition of (Abar_i, bbar_i) = (A + B K, B k + c), i = 0..N, of the last solve
//   k_seg_prefix   dx_s = F_{r-1} o ... o F_0 (dx0)
// User layouts (unpadded, row-major, per instance): summary [A (n x n), C (n x n), P (n x n), b (n),
// p (n)] = 3 n^2 + 2 n values; forward map [Phi (n x n), phi (n)] = n^2 + n values.
#pragma once

#include "lq.cuh"

namespace pdilqr {

template <typename T, int NX>
__device__ __forceinline__ void seg_load_user_elem(T *dst, const T *src, int n, int lane, int WS, unsigned mask) {
    // user summary (unpadded) -> padded VE<NX> element in shared memory (zero padding)
    using L = VE<NX>;
    for (int t = lane; t < L::SIZE; t += WS) dst[t] = T(0);
    __syncwarp(mask);
    for (int t = lane; t < n * n; t += WS) {
        const int r = t / n, c = t % n;
        dst[L::A + r * NX + c] = src[t];
        dst[L::C + r * NX + c] = src[n * n + t];
        dst[L::P + r * NX + c] = src[2 * n * n + t];
    }
    for (int t = lane; t < n; t += WS) {
        dst[L::b + t] = src[3 * n * n + t];
        dst[L::p + t] = src[3 * n * n + n + t];
    }
}

// One CTA (W workers of WS lanes) per instance; levels d = 1, 2, 4, ...: e_j <- e_j (x) e_{j+d}
// for j = 0 mod 2d, j + d <= N (in place: the right operand is never written at the same level).
template <typename T, int NX, int WS>
__global__ void __launch_bounds__(128) k_seg_reduce(int B, int N, int n, LqWork<T> ws, T *S_out) {
    using L = VE<NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int W = 128 / WS;
    const int wk = threadIdx.x / WS;
    CombineSmem<T, NX> &s = reinterpret_cast<CombineSmem<T, NX> *>(smraw)[wk];
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int b = blockIdx.x;
    if (b >= B) return;
    T *E = ws.elems + (size_t)b * (N + 2) * L::SIZE;
    __shared__ int s_fail;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int d = 1; d <= N; d <<= 1) {
        const int npairs = (N + 1 + 2 * d - 1) / (2 * d);
        for (int q = wk; q < npairs; q += W) {
            const int j = q * 2 * d;
            if (j + d > N) continue;   // odd one out: carried to the next level unchanged
            wcopy<T, L::SIZE, WS>(s.e1, E + (size_t)j * L::SIZE, lane);
            wcopy<T, L::SIZE, WS>(s.e2, E + (size_t)(j + d) * L::SIZE, lane);
            __syncwarp(mask);
            T Ao[NX], Co[NX], Po[NX], bo, po;
            const bool ok = combine_full<T, NX, WS>(s, mask, lane, Ao, Co, Po, bo, po);
            if (!ok && lane == 0) s_fail = 1;
            if (lane < NX) {
                T *o = E + (size_t)j * L::SIZE;
                st_row<T, NX, true>(o + L::A + lane * NX, Ao);
                st_row<T, NX, true>(o + L::C + lane * NX, Co);
                st_row<T, NX, true>(o + L::P + lane * NX, Po);
                o[L::b + lane] = bo;
                o[L::p + lane] = po;
            }
            __syncwarp(mask);
        }
        __syncthreads();
    }
    T *so = S_out + (size_t)b * (3 * n * n + 2 * n);
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int r = t / n, c = t % n;
        so[t] = E[L::A + r * NX + c];
        so[n * n + t] = E[L::C + r * NX + c];
        so[2 * n * n + t] = E[L::P + r * NX + c];
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        so[3 * n * n + t] = E[L::b + t];
        so[3 * n * n + n + t] = E[L::p + t];
    }
    if (threadIdx.x == 0 && s_fail) atomicMin(ws.fail + b, (1 << 24) | 1);
}

// One worker per instance: (P, p) <- cheap(S_j, (P, p)) for j = G-1 .. r+1, starting from the
// global terminal (P_term, p_term).  S_all: [G][B][3 n^2 + 2 n].
template <typename T, int NX, int WS>
__global__ void __launch_bounds__(128) k_seg_suffix(int B, int n, const T *S_all, int G, int r, const T *Pt,
                                                    const T *pt, T *P_out, T *p_out, int32_t *fail) {
    using L = VE<NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int wk = threadIdx.x / WS;
    CombineSmem<T, NX> &s = reinterpret_cast<CombineSmem<T, NX> *>(smraw)[wk];
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int b = blockIdx.x * (blockDim.x / WS) + wk;
    if (b >= B) return;
    for (int t = lane; t < L::SIZE; t += WS) s.e2[t] = T(0);
    __syncwarp(mask);
    for (int t = lane; t < n * n; t += WS) s.e2[L::P + (t / n) * NX + t % n] = Pt[(size_t)b * n * n + t];
    for (int t = lane; t < n; t += WS) s.e2[L::p + t] = pt[(size_t)b * n + t];
    __syncwarp(mask);
    bool okall = true;
    for (int j = G - 1; j > r; --j) {
        seg_load_user_elem<T, NX>(s.e1, S_all + ((size_t)j * B + b) * (3 * n * n + 2 * n), n, lane, WS, mask);
        __syncwarp(mask);
        T Po[NX], po;
        okall = combine_cheap<T, NX, WS>(s, mask, lane, Po, po) && okall;
        __syncwarp(mask);
        if (lane < NX) {
            st_row<T, NX, true>(s.e2 + L::P + lane * NX, Po);
            s.e2[L::p + lane] = po;
        }
        __syncwarp(mask);
    }
    for (int t = lane; t < n * n; t += WS) P_out[(size_t)b * n * n + t] = s.e2[L::P + (t / n) * NX + t % n];
    for (int t = lane; t < n; t += WS) p_out[(size_t)b * n + t] = s.e2[L::p + t];
    if (!okall && lane == 0) atomicMin(fail + b, (1 << 24) | 1);
}

// One worker per instance: (Phi, phi) <- (Abar_i Phi, Abar_i phi + bbar_i), i = 0..N, with the
// closed-loop elements Abar_i = A_i + B_i K_i, bbar_i = B_i k_i + c_i (Eq. 14) formed from the user's
// A, B, c and the policy K_i, k_i of the last solve (ws.Kk; the forward scans reuse ws.tel as scan
// storage, so it does not hold Abar after a solve).  F_out: [B][n^2 + n].
template <typename T, int NX, int WS>
__global__ void __launch_bounds__(128) k_seg_forward(int B, int N, int n, int m, LqArgs<T> qp, LqWork<T> ws, T *F_out) {
    using KL = KE<NX, NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int wk = threadIdx.x / WS;
    T *Ph = reinterpret_cast<T *>(smraw) + (size_t)wk * (NX * NX + NX);
    T *ph = Ph + NX * NX;
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int b = blockIdx.x * (blockDim.x / WS) + wk;
    if (b >= B) return;
    const int r = lane < n ? lane : 0;
    for (int t = lane; t < NX * NX; t += WS) Ph[t] = (t / NX == t % NX) ? T(1) : T(0);
    for (int t = lane; t < NX; t += WS) ph[t] = T(0);
    __syncwarp(mask);
    for (int i = 0; i <= N; ++i) {
        const size_t st = (size_t)b * (N + 1) + i;
        const T *A = qp.A + st * n * n, *Bm = qp.Bm + st * n * m, *c = qp.c + st * n;
        const T *Kw = ws.Kk + st * KL::SIZE;
        T arow[NX];
#pragma unroll
        for (int t = 0; t < NX; ++t) arow[t] = t < n ? A[(size_t)r * n + t] : T(0);
        T bb = c[r];
        for (int j = 0; j < m; ++j) {
            const T bj = Bm[(size_t)r * m + j];
#pragma unroll
            for (int t = 0; t < NX; ++t) arow[t] = fma(bj, Kw[KL::K + j * NX + t], arow[t]);
            bb = fma(bj, Kw[KL::k + j], bb);
        }
        T nrow[NX];
        zero(nrow);
        row_mat<T, NX, NX, NX>(nrow, arow, Ph);
        const T nph = row_dot<T, NX>(arow, ph, bb);
        __syncwarp(mask);
        if (lane < n) {
            st_row<T, NX, true>(Ph + r * NX, nrow);
            ph[r] = nph;
        }
        __syncwarp(mask);
    }
    T *fo = F_out + (size_t)b * (n * n + n);
    for (int t = lane; t < n * n; t += WS) fo[t] = Ph[(t / n) * NX + t % n];
    for (int t = lane; t < n; t += WS) fo[n * n + t] = ph[t];
}

// One worker per instance: x <- Phi_j x + phi_j for j = 0 .. r-1, x = dx0 initially.
// F_all: [G][B][n^2 + n].
template <typename T, int NX, int WS>
__global__ void __launch_bounds__(128) k_seg_prefix(int B, int n, const T *F_all, int G, int r, const T *dx0, T *dxs) {
    const int wk = threadIdx.x / WS;
    __shared__ T xs[128 / 4][NX];
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int b = blockIdx.x * (blockDim.x / WS) + wk;
    if (b >= B) return;
    T *x = xs[wk];
    for (int t = lane; t < NX; t += WS) x[t] = t < n ? dx0[(size_t)b * n + t] : T(0);
    __syncwarp(mask);
    for (int j = 0; j < r; ++j) {
        const T *F = F_all + ((size_t)j * B + b) * (n * n + n);
        T v = T(0);
        if (lane < n) {
            v = F[n * n + lane];
            for (int t = 0; t < n; ++t) v = fma(F[lane * n + t], x[t], v);
        }
        __syncwarp(mask);
        if (lane < n) x[lane] = v;
        __syncwarp(mask);
    }
    for (int t = lane; t < n; t += WS) dxs[(size_t)b * n + t] = x[t];
    (void)G;
}

}  // namespace pdilqr
