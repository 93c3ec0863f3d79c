// lq.cuh -- LQ/KKT subproblem (Eq. 4) by parallel associative scans on sm_100a.
//
// Kernels (one launch each, all stream-ordered, no host sync):
//   k_elem_init   Eq. 12 / Eq. 13 element initialisation, one worker per (instance, stage)
//   k_scan_bwd    reverse inclusive scan of value elements with the combination rule (Eq. 11,
//                 corrected: DESIGN.md readings R1, R2); chunked Blelloch tree, one CTA per instance
//   k_policy      per-stage policy K, k from the scanned P_{i+1}, p_{i+1} (Eq. 5 rows) and
//                 the closed-loop elements (Abar, bbar) of Eq. 14
//   k_scan_fwd    forward inclusive scan of the conditional optimal trajectory (Eq. 15, combine
//                 order corrected: reading R6) -> dx
//   k_tail        du = K dx + k (Eq. 6) and the dual update dlam = P dx + p (Eq. 7)
// Value element e = (A~, C~, P~, b~, p~) of Eq. 10; a "suffix" is an element whose A~ = C~ = b~ = 0
// (every product that contains the terminal element, Eq. 13), combined by the cheap rule.
#pragma once

#include <climits>

#include <cooperative_groups.h>

#include "common.cuh"

namespace pdilqr {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------------- layouts
template <int NX>
struct VE {  // value element, units of T; every field starts 16-byte aligned
    static constexpr int A = 0, C = NX * NX, P = 2 * NX * NX, b = 3 * NX * NX, p = 3 * NX * NX + NX;
    static constexpr int SIZE = 3 * NX * NX + 2 * NX;
};
template <int NX>
struct TE {  // trajectory element (Abar, bbar) of Eq. 15; also used for (P, p) and (K, k) rows
    static constexpr int A = 0, b = NX * NX, SIZE = NX * NX + NX;
};
template <int NX, int NU>
struct KE {  // policy (K, k) of one stage
    static constexpr int K = 0, k = NU * NX, SIZE = NU * NX + NU;
};

constexpr int kFailNone = 0x7f7f7f7f;  // LqWork::fail after cudaMemsetAsync(0x7f): no failure

enum SlotKind : int { SLOT_IDENT = 0, SLOT_ANCHOR = 1, SLOT_GENERAL = 2 };  // ANCHOR = suffix / anchored prefix

template <typename T>
struct LqArgs {  // user Eq. 4 data (runtime n, m strides)
    const T *A, *Bm, *c, *Q, *R, *S, *q, *r, *Pt, *pt, *dx0;
};

template <typename T>
struct LqOut {
    T *dx, *du, *dlam, *K, *k;  // user buffers (K, k may be null)
};

// Workspace views used by the LQ kernels (sizes in pdilqr.cu).
template <typename T>
struct LqWork {
    T *elems;    // [B][N+2][VE]
    T *vslots;   // [B][Pv][VE]      (tree slots of the backward scan)
    T *Pp;       // [B][N+2][TE]      P_i, p_i
    T *Kk;       // [B][N+1][KE]      K_i, k_i
    T *tel;      // [B][N+1][TE]      Abar_i, bbar_i
    T *tslots;   // [B][Pf][TE]       tree slots of the forward scan
    T *dxw;      // [B][N+2][NX]      dx (padded)
    int32_t *fail;    // [B] min(stage+1) of a failed factorisation, kFailNone if none
    int32_t *nonfin;  // [B] non-finite output flag
};

// Cooperative copy of NV values (16-byte granules) by one worker.
template <typename T, int NV, int WS>
__device__ __forceinline__ void wcopy(T *__restrict__ dst, const T *__restrict__ src, int lane) {
    static_assert((NV * sizeof(T)) % 16 == 0, "granule");
    constexpr int NG = NV * sizeof(T) / 16;
    const int4 *s = reinterpret_cast<const int4 *>(src);
    int4 *d = reinterpret_cast<int4 *>(dst);
#pragma unroll 4
    for (int i = lane; i < NG; i += WS) d[i] = s[i];
}
template <typename T, int NV, int WS>
__device__ __forceinline__ void wzero(T *__restrict__ dst, int lane) {
    constexpr int NG = NV * sizeof(T) / 16;
    int4 *d = reinterpret_cast<int4 *>(dst);
    for (int i = lane; i < NG; i += WS) d[i] = make_int4(0, 0, 0, 0);
}

// ------------------------------------------------------------------------- value combines
// Symmetrise a row-distributed matrix through shared scratch: out[r][j] = (M[r][j] + M[j][r]) / 2.
// P~ and C~ are symmetric in exact arithmetic (SPEC S:76 re-symmetrisation); without this, rounding
// asymmetry accumulates along the scan.
template <typename T, int NX>
__device__ __forceinline__ void symmetrize_rows(T (&row)[NX], T *scratch, unsigned mask, int lane) {
    const int r = lane < NX ? lane : 0;
    if (lane < NX) st_row<T, NX, true>(scratch + r * NX, row);
    __syncwarp(mask);
    T col[NX];
    ld_col<T, NX>(col, scratch + r, NX);
#pragma unroll
    for (int j = 0; j < NX; ++j) row[j] = T(0.5) * (row[j] + col[j]);
    __syncwarp(mask);
}

template <typename T, int NX>
struct CombineSmem {
    T e1[VE<NX>::SIZE];  // left operand  e_{i->k}
    T e2[VE<NX>::SIZE];  // right operand e_{k->j}
    T X[NX * NX], Y[NX * NX], V[NX * NX];
    T z[NX], w[NX];
};

// Full combination rule e1 (x) e2 (Eq. 11 as corrected in SURVEY App. A / DESIGN.md R1-R2):
//   M = I + C1 P2 (pivoted Gauss-Jordan), X = M^-1 A1, Y = M^-1 C1, z = M^-1 (b1 - C1 p2)
//   A = A2 X, b = A2 z + b2, C = A2 Y A2^T + C2, P = A1^T P2 X + P1,
//   p = A1^T M^-T w + p1 = X^T w + p1,  w = p2 + P2 b1
// Operands in smem (s.e1, s.e2); lane r < NX returns row r of A, C, P and b_r, p_r.
template <typename T, int NX, int WS>
__device__ __forceinline__ bool combine_full(CombineSmem<T, NX> &s, unsigned mask, int lane, T (&Ao)[NX],
                                             T (&Co)[NX], T (&Po)[NX], T &bo, T &po) {
    using L = VE<NX>;
    const int r = lane < NX ? lane : 0;
    T c1[NX];
    ld_row<T, NX, true>(c1, s.e1 + L::C + r * NX);
    T M[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) M[j] = (j == r) ? T(1) : T(0);
    row_mat<T, NX, NX, NX>(M, c1, s.e2 + L::P);
    T rhs[2 * NX + 1];
    {
        T a1[NX];
        ld_row<T, NX, true>(a1, s.e1 + L::A + r * NX);
#pragma unroll
        for (int j = 0; j < NX; ++j) { rhs[j] = a1[j]; rhs[NX + j] = c1[j]; }
        rhs[2 * NX] = s.e1[L::b + r] - row_dot<T, NX>(c1, s.e2 + L::p, T(0));
    }
    int pr;
    const bool ok = gauss_jordan<T, WS, NX, 2 * NX + 1, true>(mask, M, rhs, lane, NX, pr);
    if (pr >= 0) {
        T xr[NX], yr[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) { xr[j] = rhs[j]; yr[j] = rhs[NX + j]; }
        st_row<T, NX, true>(s.X + pr * NX, xr);
        st_row<T, NX, true>(s.Y + pr * NX, yr);
        s.z[pr] = rhs[2 * NX];
    }
    __syncwarp(mask);
    T a2[NX];
    ld_row<T, NX, true>(a2, s.e2 + L::A + r * NX);
    zero(Ao);
    row_mat<T, NX, NX, NX>(Ao, a2, s.X);
    bo = row_dot<T, NX>(a2, s.z, s.e2[L::b + r]);
    {
        T W[NX];
        zero(W);
        row_mat<T, NX, NX, NX>(W, a2, s.Y);
        ld_row<T, NX, true>(Co, s.e2 + L::C + r * NX);
        row_matT<T, NX, NX, NX>(Co, W, s.e2 + L::A);
    }
    T p2[NX];
    ld_row<T, NX, true>(p2, s.e2 + L::P + r * NX);
    T wr;
    {
        T V[NX];
        zero(V);
        row_mat<T, NX, NX, NX>(V, p2, s.X);
        wr = row_dot<T, NX>(p2, s.e1 + L::b, s.e2[L::p + r]);
        if (lane < NX) { st_row<T, NX, true>(s.V + r * NX, V); s.w[r] = wr; }
    }
    __syncwarp(mask);
    T a1c[NX];
    ld_col<T, NX>(a1c, s.e1 + L::A + r, NX);
    ld_row<T, NX, true>(Po, s.e1 + L::P + r * NX);
    row_mat<T, NX, NX, NX>(Po, a1c, s.V);
    // p = A1^T M^-T w + p1 = X^T w + p1  (A1^T M^-T = (M^-1 A1)^T: no I - P2 M^-1 C1 cancellation)
    {
        T xc[NX];
        ld_col<T, NX>(xc, s.X + r, NX);
        po = row_dot<T, NX>(xc, s.w, s.e1[L::p + r]);
    }
    __syncwarp(mask);
    symmetrize_rows<T, NX>(Po, s.V, mask, lane);
    symmetrize_rows<T, NX>(Co, s.Y, mask, lane);
    return ok;
}

// Cheap rule for a suffix right operand (A2 = C2 = b2 = 0): only P, p of the result are nonzero.
//   X = M^-1 A1 (M = I + C1 P2),  P = A1^T P2 X + P1,  p = X^T (p2 + P2 b1) + p1.
template <typename T, int NX, int WS>
__device__ __forceinline__ bool combine_cheap(CombineSmem<T, NX> &s, unsigned mask, int lane, T (&Po)[NX], T &po) {
    using L = VE<NX>;
    const int r = lane < NX ? lane : 0;
    T M[NX];
    {
        T c1[NX];
        ld_row<T, NX, true>(c1, s.e1 + L::C + r * NX);
#pragma unroll
        for (int j = 0; j < NX; ++j) M[j] = (j == r) ? T(1) : T(0);
        row_mat<T, NX, NX, NX>(M, c1, s.e2 + L::P);
    }
    T p2[NX];
    ld_row<T, NX, true>(p2, s.e2 + L::P + r * NX);
    const T wr = row_dot<T, NX>(p2, s.e1 + L::b, s.e2[L::p + r]);
    if (lane < NX) s.w[r] = wr;
    T rhs[NX];
    ld_row<T, NX, true>(rhs, s.e1 + L::A + r * NX);
    int pr;
    const bool ok = gauss_jordan<T, WS, NX, NX, true>(mask, M, rhs, lane, NX, pr);
    if (pr >= 0) st_row<T, NX, true>(s.X + pr * NX, rhs);
    __syncwarp(mask);
    {
        T V[NX];
        zero(V);
        row_mat<T, NX, NX, NX>(V, p2, s.X);
        if (lane < NX) st_row<T, NX, true>(s.V + r * NX, V);
    }
    T xc[NX];
    ld_col<T, NX>(xc, s.X + r, NX);
    po = row_dot<T, NX>(xc, s.w, s.e1[L::p + r]);
    __syncwarp(mask);
    T a1c[NX];
    ld_col<T, NX>(a1c, s.e1 + L::A + r, NX);
    ld_row<T, NX, true>(Po, s.e1 + L::P + r * NX);
    row_mat<T, NX, NX, NX>(Po, a1c, s.V);
    __syncwarp(mask);
    symmetrize_rows<T, NX>(Po, s.Y, mask, lane);
    return ok;
}

// ------------------------------------------------------------------ element init (Eq. 12-13)
// Per stage i <= N:  GJ on R (SPD, no pivoting) with right-hand sides [S | r | B^T], then
//   A~ = A - B R^-1 S,  C~ = B R^-1 B^T,  b~ = b - B R^-1 r,  P~ = Q - S^T R^-1 S,  p~ = q - S^T R^-1 r.
// Terminal element i = N+1 (Eq. 13, reading R4): A~ = C~ = b~ = 0, P~ = P_{N+1}, p~ = p_{N+1}.
// Padded instantiations (n < NX or m < NU): state rows/cols >= n are zero, R is padded with
// the identity; the padded entries of every element are then exactly zero.
// Per-worker shared memory words of k_elem_init: ZS, ZB, zr; the exact instantiation also stages the
// stage's R, S, B, A, Q, r, c, q there with one cp.async burst (all global loads in flight at once
// instead of two dependent load phases around the elimination; ncu r2_elem: the kernel was bound by
// global-load latency, long-scoreboard 2.7 per issue at 8 warps per SM).
template <int NX, int NU, bool EX>
__host__ __device__ constexpr int elem_init_smw() {
    return 2 * NU * NX + round_up4(NU) + (EX ? 5 * NX * NX + 3 * NX : 0);
}

template <typename T, int NX, int NU, bool EX>
__global__ void __launch_bounds__(128, (sizeof(T) == 4 && NX <= 12) ? 3 : 1) k_elem_init(LqArgs<T> qp, int B, int N, int n, int m, LqWork<T> ws) {
    constexpr int WS = worker_width(NX > NU ? NX : NU);
    constexpr int SMW = elem_init_smw<NX, NU, EX>();
    using L = VE<NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int wloc = threadIdx.x / WS;
    const long gw = (long)blockIdx.x * (blockDim.x / WS) + wloc;
    const int L2 = N + 2;
    if (gw >= (long)B * L2) return;  // whole worker exits together
    const int b = (int)(gw / L2), i = (int)(gw % L2);
    T *sm = reinterpret_cast<T *>(smraw) + wloc * SMW;
    T *ZS = sm, *ZB = sm + NU * NX, *zr = sm + 2 * NU * NX;
    T *e = ws.elems + ((size_t)b * L2 + i) * L::SIZE;
    const int r = lane < NX ? lane : 0;
    if (i == N + 1) {  // terminal element
        if (lane < NX) {
            T zrow[NX], prow[NX];
            zero(zrow);
            if (EX || r < n) ld_row<T, NX, EX>(prow, qp.Pt + (size_t)b * n * n + r * n, n);
            else zero(prow);
            st_row<T, NX, true>(e + L::A + r * NX, zrow);
            st_row<T, NX, true>(e + L::C + r * NX, zrow);
            st_row<T, NX, true>(e + L::P + r * NX, prow);
            e[L::b + r] = T(0);
            e[L::p + r] = (EX || r < n) ? qp.pt[(size_t)b * n + r] : T(0);
        }
        return;
    }
    const size_t st = (size_t)b * (N + 1) + i;
    // exact instantiation: the stage's R, S, B, A, Q (NX x NX each) and r, c, q into shared memory,
    // 16-byte cp.async chunks spread over the worker's lanes, one wait
    T *stg = sm + 2 * NU * NX + round_up4(NU);
    const T *gR = qp.R + st * m * m, *gS = qp.S + st * m * n, *gB = qp.Bm + st * n * m;
    const T *gA = qp.A + st * n * n, *gQ = qp.Q + st * n * n;
    if constexpr (EX) {
        constexpr int EPC = 16 / (int)sizeof(T), MC = NX * NX / EPC, VC = NX / EPC;
        for (int ch = lane; ch < 5 * MC + 3 * VC; ch += WS) {
            if (ch < 5 * MC) {
                const int am = ch / MC, k = (ch - am * MC) * EPC;
                const T *src = am == 0 ? gR : am == 1 ? gS : am == 2 ? gB : am == 3 ? gA : gQ;
                cp_async16(stg + am * NX * NX + k, src + k);
            } else {
                const int av = (ch - 5 * MC) / VC, k = (ch - 5 * MC - av * VC) * EPC;
                const T *src = av == 0 ? qp.r + st * m : av == 1 ? qp.c + st * n : qp.q + st * n;
                cp_async16(stg + 5 * NX * NX + av * NX + k, src + k);
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp(mask);
        gR = stg; gS = stg + NX * NX; gB = stg + 2 * NX * NX; gA = stg + 3 * NX * NX; gQ = stg + 4 * NX * NX;
    }
    const T *vr_ = EX ? stg + 5 * NX * NX : qp.r + st * m;
    const T *vc_ = EX ? stg + 5 * NX * NX + NX : qp.c + st * n;
    const T *vq_ = EX ? stg + 5 * NX * NX + 2 * NX : qp.q + st * n;
    // --- GJ rows: lane r < NU owns row r of R and of [S | r | B^T]
    {
        const int ru = lane < NU ? lane : 0;
        T a[NU], rhs[2 * NX + 1];
        const bool valid = EX || ru < m;
        if (valid) {
            ld_row<T, NU, EX>(a, gR + ru * m, m);
            T srow[NX], bcol[NX];
            ld_row<T, NX, EX>(srow, gS + ru * n, n);
            ld_col<T, NX>(bcol, gB + ru, m, n);
#pragma unroll
            for (int j = 0; j < NX; ++j) { rhs[j] = srow[j]; rhs[NX + 1 + j] = bcol[j]; }
            rhs[NX] = vr_[ru];
        } else {
#pragma unroll
            for (int j = 0; j < NU; ++j) a[j] = (j == ru) ? T(1) : T(0);
#pragma unroll
            for (int j = 0; j < 2 * NX + 1; ++j) rhs[j] = T(0);
        }
        int pr;
        const bool ok = gauss_jordan<T, WS, NU, 2 * NX + 1, false>(mask, a, rhs, lane, NU, pr);
        if (!ok && lane == 0) atomicMin(ws.fail + b, i + 1);
        if (pr >= 0) {
            T t1[NX], t2[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) { t1[j] = rhs[j]; t2[j] = rhs[NX + 1 + j]; }
            st_row<T, NX, true>(ZS + pr * NX, t1);
            st_row<T, NX, true>(ZB + pr * NX, t2);
            zr[pr] = rhs[NX];
        }
    }
    __syncwarp(mask);
    // --- element rows: lane r < NX owns state row r
    T brow[NU], scol[NU], row[NX], out[NX];
    const bool vr = EX || r < n;
    if (vr) {
        ld_row<T, NU, EX>(brow, gB + r * m, m);
        ld_col<T, NU>(scol, gS + r, n, m);
    } else {
        zero(brow);
        zero(scol);
    }
    // A~
    if (vr) ld_row<T, NX, EX>(row, gA + r * n, n);
    else zero(row);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
        T y[NX];
        ld_row<T, NX, true>(y, ZS + k * NX);
#pragma unroll
        for (int j = 0; j < NX; ++j) row[j] = fma(-brow[k], y[j], row[j]);
    }
    if (lane < NX) st_row<T, NX, true>(e + L::A + r * NX, row);
    // C~ = B (R^-1 B^T)
    zero(out);
    row_mat<T, NU, NX, NX>(out, brow, ZB);
    if (lane < NX) st_row<T, NX, true>(e + L::C + r * NX, out);
    // P~ = Q - S^T (R^-1 S)
    if (vr) ld_row<T, NX, EX>(row, gQ + r * n, n);
    else zero(row);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
        T y[NX];
        ld_row<T, NX, true>(y, ZS + k * NX);
#pragma unroll
        for (int j = 0; j < NX; ++j) row[j] = fma(-scol[k], y[j], row[j]);
    }
    if (lane < NX) st_row<T, NX, true>(e + L::P + r * NX, row);
    const T cb = vr ? vc_[r] : T(0);
    const T qq = vr ? vq_[r] : T(0);
    T bt = cb, pt = qq;
#pragma unroll
    for (int k = 0; k < NU; ++k) { bt = fma(-brow[k], zr[k], bt); pt = fma(-scol[k], zr[k], pt); }
    if (lane < NX) { e[L::b + r] = bt; e[L::p + r] = pt; }
}

// Element initialisation for exact 12 x 12 problems with TWO ROWS PER LANE (design D11 of the
// fused fold applied to Eq. 12): a worker is 6 lanes, lane l owns rows l and l + 6, 4 items (instance,
// stage) per warp (lanes 24-31 shadow lane 23 and store nothing).  The stage's R, S, B, A, Q, r, c, q
// arrive in one cp.async burst; the SPD Gauss-Jordan on R with the 25 right-hand sides [S | r | B^T]
// keeps both rows of a lane in one FFMA2; then A~ = A - B Z_S, C~ = B Z_B, P~ = Q - S^T Z_S,
// b~ = c - B z_r, p~ = q - S^T z_r with every loaded operand row feeding two row updates.  A terminal
// item (i = N+1) runs the same code on R = I and then writes Eq. 13 instead (the warp's shuffles stay
// converged).  Same arithmetic as k_elem_init.
template <typename T>
struct ElemR2Smem {
    T R[144], S[144], Bm[144], A[144], Q[144], r[12], c[12], q[12];
    T ZS[144], ZB[144], zr[12];
    T pad[8];
};

template <typename T>
__global__ void __launch_bounds__(64) k_elem_init_r2(LqArgs<T> qp, int B, int N, LqWork<T> ws) {
    constexpr int NX = 12, NW = 4, NL = 6 * NW, NRHS = 2 * NX + 1;
    using L = VE<NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int Ln = threadIdx.x & 31;
    const int w = Ln < NL ? Ln / 6 : NW - 1;
    const int l = Ln < NL ? Ln - 6 * w : 5;
    const bool lane_act = Ln < NL;
    ElemR2Smem<T> &s = reinterpret_cast<ElemR2Smem<T> *>(smraw)[(threadIdx.x >> 5) * NW + w];
    const int L2 = N + 2;
    const long total = (long)B * L2;
    const long item_raw = ((long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NW + w;
    if (__all_sync(0xffffffffu, item_raw >= total)) return;
    const bool live = item_raw < total;
    const long item = live ? item_raw : total - 1;
    const int b = (int)(item / L2), i = (int)(item - (long)b * L2);
    const bool term = i == N + 1;
    const bool act = lane_act && live;
    const int r0 = l, r1 = l + 6, wb = 6 * w;
    const size_t st = (size_t)b * (N + 1) + (term ? 0 : i);
    // ---- stage inputs (a terminal item uses R = I and zeros: same elimination, result discarded)
    if (!term) {
        constexpr int EPC = 16 / (int)sizeof(T), MC = NX * NX / EPC, VC = NX / EPC;
        if (lane_act) {
            for (int ch = l; ch < 5 * MC + 3 * VC; ch += 6) {
                if (ch < 5 * MC) {
                    const int am = ch / MC, k = (ch - am * MC) * EPC;
                    const T *src = am == 0 ? qp.R + st * 144 : am == 1 ? qp.S + st * 144 : am == 2 ? qp.Bm + st * 144
                                 : am == 3 ? qp.A + st * 144 : qp.Q + st * 144;
                    cp_async16(s.R + am * 144 + k, src + k);
                } else {
                    const int av = (ch - 5 * MC) / VC, k = (ch - 5 * MC - av * VC) * EPC;
                    const T *src = av == 0 ? qp.r + st * 12 : av == 1 ? qp.c + st * 12 : qp.q + st * 12;
                    cp_async16(s.r + av * 12 + k, src + k);
                }
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
    } else if (lane_act) {
        for (int t = l; t < 5 * 144 + 36; t += 6) s.R[t] = (t < 144 && t % 13 == 0) ? T(1) : T(0);
    }
    __syncwarp();
    // ---- SPD Gauss-Jordan: lane l holds rows l, l + 6 of R and of [S | r | B^T]
    T a0[NX], a1[NX], x0[NRHS], x1[NRHS];
    ld_row<T, NX, true>(a0, s.R + r0 * NX);
    ld_row<T, NX, true>(a1, s.R + r1 * NX);
    {
        T t0[NX], t1[NX];
        ld_row<T, NX, true>(t0, s.S + r0 * NX);
        ld_row<T, NX, true>(t1, s.S + r1 * NX);
#pragma unroll
        for (int j = 0; j < NX; ++j) { x0[j] = t0[j]; x1[j] = t1[j]; }
        x0[NX] = s.r[r0];
        x1[NX] = s.r[r1];
#pragma unroll
        for (int j = 0; j < NX; ++j) { x0[NX + 1 + j] = s.Bm[j * NX + r0]; x1[NX + 1 + j] = s.Bm[j * NX + r1]; }
    }
    bool ok = true;
    T piv0 = T(1), piv1 = T(1);
#pragma unroll
    for (int k = 0; k < NX; ++k) {
        const int pl = k % 6, ps = k / 6;
        const int src = wb + pl;
        const T own = ps == 0 ? a0[k] : a1[k];
        const T rk = rcp_rn(own);
        const T pvv = __shfl_sync(0xffffffffu, own, src);
        const T rpv = __shfl_sync(0xffffffffu, rk, src);
        ok = ok && (pvv > T(0)) && isfinite(pvv);
        const bool isp0 = ps == 0 && l == pl, isp1 = ps == 1 && l == pl;
        const T f0 = isp0 ? T(0) : a0[k] * rpv;
        const T f1 = isp1 ? T(0) : a1[k] * rpv;
        if (isp0) piv0 = pvv;
        if (isp1) piv1 = pvv;
#pragma unroll
        for (int j = k + 1; j < NX; ++j) {
            const T pj = __shfl_sync(0xffffffffu, ps == 0 ? a0[j] : a1[j], src);
            ffma2(-f0, -f1, pj, pj, a0[j], a1[j]);
        }
#pragma unroll
        for (int j = 0; j < NRHS; ++j) {
            const T pj = __shfl_sync(0xffffffffu, ps == 0 ? x0[j] : x1[j], src);
            ffma2(-f0, -f1, pj, pj, x0[j], x1[j]);
        }
    }
    {
        const T i0 = rcp_rn(piv0), i1 = rcp_rn(piv1);
#pragma unroll
        for (int j = 0; j < NRHS; ++j) { x0[j] *= i0; x1[j] *= i1; }
    }
    if (!term && !ok && l == 0 && act) atomicMin(ws.fail + b, i + 1);
    if (lane_act) {   // Z_S, z_r, Z_B rows (all lanes of live and shadow workers write their own slice)
        T zs0[NX], zs1[NX], zb0[NX], zb1[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) { zs0[j] = x0[j]; zs1[j] = x1[j]; zb0[j] = x0[NX + 1 + j]; zb1[j] = x1[NX + 1 + j]; }
        st_row<T, NX, true>(s.ZS + r0 * NX, zs0);
        st_row<T, NX, true>(s.ZS + r1 * NX, zs1);
        st_row<T, NX, true>(s.ZB + r0 * NX, zb0);
        st_row<T, NX, true>(s.ZB + r1 * NX, zb1);
        s.zr[r0] = x0[NX];
        s.zr[r1] = x1[NX];
    }
    __syncwarp();
    T *e = ws.elems + ((size_t)b * L2 + i) * L::SIZE;
    if (term) {   // Eq. 13: A~ = C~ = 0, P~ = P_{N+1}, b~ = 0, p~ = p_{N+1}
        if (act) {
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
                const int r = l + 6 * sl;
                T z[NX], pr[NX];
                zero(z);
                ld_row<T, NX, true>(pr, qp.Pt + (size_t)b * 144 + r * NX);
                st_row<T, NX, true>(e + L::A + r * NX, z);
                st_row<T, NX, true>(e + L::C + r * NX, z);
                st_row<T, NX, true>(e + L::P + r * NX, pr);
                e[L::b + r] = T(0);
                e[L::p + r] = qp.pt[(size_t)b * NX + r];
            }
        }
        return;
    }
    // ---- element rows r0, r1
    T br0[NX], br1[NX], sc0[NX], sc1[NX];
    ld_row<T, NX, true>(br0, s.Bm + r0 * NX);
    ld_row<T, NX, true>(br1, s.Bm + r1 * NX);
#pragma unroll
    for (int k = 0; k < NX; ++k) { sc0[k] = s.S[k * NX + r0]; sc1[k] = s.S[k * NX + r1]; }
    {   // A~ = A - B Z_S
        T o0[NX], o1[NX];
        ld_row<T, NX, true>(o0, s.A + r0 * NX);
        ld_row<T, NX, true>(o1, s.A + r1 * NX);
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            T y[NX];
            ld_row<T, NX, true>(y, s.ZS + k * NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) ffma2(-br0[k], -br1[k], y[j], y[j], o0[j], o1[j]);
        }
        if (act) { st_row<T, NX, true>(e + L::A + r0 * NX, o0); st_row<T, NX, true>(e + L::A + r1 * NX, o1); }
    }
    {   // C~ = B Z_B
        T o0[NX], o1[NX];
        zero(o0);
        zero(o1);
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            T y[NX];
            ld_row<T, NX, true>(y, s.ZB + k * NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) ffma2(br0[k], br1[k], y[j], y[j], o0[j], o1[j]);
        }
        if (act) { st_row<T, NX, true>(e + L::C + r0 * NX, o0); st_row<T, NX, true>(e + L::C + r1 * NX, o1); }
    }
    {   // P~ = Q - S^T Z_S
        T o0[NX], o1[NX];
        ld_row<T, NX, true>(o0, s.Q + r0 * NX);
        ld_row<T, NX, true>(o1, s.Q + r1 * NX);
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            T y[NX];
            ld_row<T, NX, true>(y, s.ZS + k * NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) ffma2(-sc0[k], -sc1[k], y[j], y[j], o0[j], o1[j]);
        }
        if (act) { st_row<T, NX, true>(e + L::P + r0 * NX, o0); st_row<T, NX, true>(e + L::P + r1 * NX, o1); }
    }
    T bt0 = s.c[r0], bt1 = s.c[r1], pt0 = s.q[r0], pt1 = s.q[r1];
#pragma unroll
    for (int k = 0; k < NX; ++k) {
        const T z = s.zr[k];
        ffma2(-br0[k], -br1[k], z, z, bt0, bt1);
        ffma2(-sc0[k], -sc1[k], z, z, pt0, pt1);
    }
    if (act) { e[L::b + r0] = bt0; e[L::b + r1] = bt1; e[L::p + r0] = pt0; e[L::p + r1] = pt1; }
}

// Negative control of the parity tests (PDILQR_FAULT_COMBINE=1, never set in
// production): perturb P~[0][0] of the element of stage floor(N/2) of instance 0 by 1e-3 (1 + |P~00|),
// so every combine that consumes it is wrong; the parity tests must then fail for instance 0.
template <typename T, int NX>
__global__ void k_fault_inject(LqWork<T> ws, int N) {
    T *e = ws.elems + (size_t)(N / 2) * VE<NX>::SIZE + VE<NX>::P;
    e[0] += T(1e-3) * (T(1) + fabs(e[0]));
}

// -------------------------------------------------------------------- backward scan (Eq. 8-11)
// One CTA per instance, W workers.  L = N+2 elements are cut into J = ceil(L / chunk) chunks.
//  phase 1: every chunk j < J-1 is reduced right-to-left into its summary S_j by the full rule;
//           the last chunk (it holds the terminal element) is folded right-to-left by the cheap
//           rule, which yields its final suffixes s_i = e_i (x) ... (x) e_{N+1} directly;
//  phase 2: exclusive suffix products T_j = S_{j+1} (x) ... (x) S_{J-1} by a work-efficient
//           Blelloch tree (up-sweep / down-sweep, 2 ceil(log2 J) levels) on the reversed slots;
//  phase 3: every chunk j < J-1 is folded right-to-left from T_j by the cheap rule.
// Read-out (reading R5): P_i = P~(s_i), p_i = p~(s_i), i = 0..N+1.
// chunk = 1 is the pure tree over all elements (the paper's scan); chunk >= L the pure fold.
template <typename T, int NX>
struct ScanBwd {
    static constexpr int WS = worker_width(NX);
    using L = VE<NX>;

    static __device__ __forceinline__ void store_elem_rows(T *dst, const T (&A)[NX], const T (&C)[NX],
                                                           const T (&P)[NX], T b, T p, int lane) {
        if (lane < NX) {
            st_row<T, NX, true>(dst + L::A + lane * NX, A);
            st_row<T, NX, true>(dst + L::C + lane * NX, C);
            st_row<T, NX, true>(dst + L::P + lane * NX, P);
            dst[L::b + lane] = b;
            dst[L::p + lane] = p;
        }
    }
    static __device__ __forceinline__ void store_suffix_rows(T *dst, const T (&P)[NX], T p, int lane) {
        if (lane < NX) {
            T z[NX];
            zero(z);
            st_row<T, NX, true>(dst + L::A + lane * NX, z);
            st_row<T, NX, true>(dst + L::C + lane * NX, z);
            st_row<T, NX, true>(dst + L::P + lane * NX, P);
            dst[L::b + lane] = T(0);
            dst[L::p + lane] = p;
        }
    }
    // write (P, p) of suffix s_i to the value-function buffer
    static __device__ __forceinline__ void out_Pp(T *Pp_i, const T (&P)[NX], T p, int lane) {
        if (lane < NX) {
            st_row<T, NX, true>(Pp_i + lane * NX, P);
            Pp_i[NX * NX + lane] = p;
        }
    }
};

// Work units of the backward scan (one worker each).  Operands are staged from global memory
// (L2) into the worker's shared slice; results go back to global memory.  `kind` holds the slot
// kinds of one instance (identity / suffix / general).
template <typename T, int NX>
struct BwdUnits {
    using SB = ScanBwd<T, NX>;
    using L = VE<NX>;
    static constexpr int WS = SB::WS;
    static constexpr int TP = TE<NX>::SIZE;

    // phase 1: chunk j = [j c, min((j+1) c, L)) reduced right-to-left (the last chunk holds the
    // terminal element and is folded with the cheap rule, writing its final suffixes).
    static __device__ void phase1(CombineSmem<T, NX> &s, unsigned mask, int lane, const T *E, T *Y, int *kind, T *Pp,
                                  int j, int chunk, int J, int L2, int &fail) {
        const int lo = j * chunk, hi = min(lo + chunk, L2);
        wcopy<T, L::SIZE, WS>(s.e2, E + (size_t)(hi - 1) * L::SIZE, lane);
        __syncwarp(mask);
        if (j == J - 1) {
            if (lane < NX) {
                T P[NX];
                ld_row<T, NX, true>(P, s.e2 + L::P + lane * NX);
                SB::out_Pp(Pp + (size_t)(hi - 1) * TP, P, s.e2[L::p + lane], lane);
            }
            for (int i = hi - 2; i >= lo; --i) {
                wcopy<T, L::SIZE, WS>(s.e1, E + (size_t)i * L::SIZE, lane);
                __syncwarp(mask);
                T Po[NX], po;
                if (!combine_cheap<T, NX, WS>(s, mask, lane, Po, po)) fail = min(fail, i + 1);
                if (lane < NX) {
                    st_row<T, NX, true>(s.e2 + L::P + lane * NX, Po);
                    s.e2[L::p + lane] = po;
                }
                SB::out_Pp(Pp + (size_t)i * TP, Po, po, lane);
                __syncwarp(mask);
            }
            if (J > 1) {
                T P[NX];
                ld_row<T, NX, true>(P, s.e2 + L::P + (lane < NX ? lane : 0) * NX);
                SB::store_suffix_rows(Y, P, s.e2[L::p + (lane < NX ? lane : 0)], lane);
                if (lane == 0) kind[0] = SLOT_ANCHOR;
            }
        } else {
            for (int i = hi - 2; i >= lo; --i) {
                wcopy<T, L::SIZE, WS>(s.e1, E + (size_t)i * L::SIZE, lane);
                __syncwarp(mask);
                T Ao[NX], Co[NX], Po[NX], bo, po;
                if (!combine_full<T, NX, WS>(s, mask, lane, Ao, Co, Po, bo, po)) fail = min(fail, i + 1);
                SB::store_elem_rows(s.e2, Ao, Co, Po, bo, po, lane);
                __syncwarp(mask);
            }
            wcopy<T, L::SIZE, WS>(Y + (size_t)(J - 1 - j) * L::SIZE, s.e2, lane);
            if (lane == 0) kind[J - 1 - j] = SLOT_GENERAL;
        }
        __syncwarp(mask);
    }
    // phase 2 up-sweep node k (level d) on the reversed slots: Y[k] = Y[k] (x) Y[k-d]
    static __device__ void up(CombineSmem<T, NX> &s, unsigned mask, int lane, T *Y, int *kind, int k, int d, int &fail) {
        const int kr = k - d;
        const int kl_kind = kind[k], kr_kind = kind[kr];
        __syncwarp(mask);
        T *Yk = Y + (size_t)k * L::SIZE, *Yr = Y + (size_t)kr * L::SIZE;
        if (kr_kind == SLOT_IDENT) {
        } else if (kl_kind == SLOT_IDENT) {
            wcopy<T, L::SIZE, WS>(Yk, Yr, lane);
            if (lane == 0) kind[k] = kr_kind;
        } else {
            wcopy<T, L::SIZE, WS>(s.e1, Yk, lane);
            wcopy<T, L::SIZE, WS>(s.e2, Yr, lane);
            __syncwarp(mask);
            if (kr_kind == SLOT_ANCHOR) {
                T Po[NX], po;
                if (!combine_cheap<T, NX, WS>(s, mask, lane, Po, po)) fail = min(fail, 1);
                SB::store_suffix_rows(Yk, Po, po, lane);
                if (lane == 0) kind[k] = SLOT_ANCHOR;
            } else {
                T Ao[NX], Co[NX], Po[NX], bo, po;
                if (!combine_full<T, NX, WS>(s, mask, lane, Ao, Co, Po, bo, po)) fail = min(fail, 1);
                SB::store_elem_rows(Yk, Ao, Co, Po, bo, po, lane);
            }
        }
        __syncwarp(mask);
    }
    // phase 2 down-sweep node k (level d): t = Y[k-d]; Y[k-d] = Y[k]; Y[k] = t (x) Y[k]
    static __device__ void down(CombineSmem<T, NX> &s, unsigned mask, int lane, T *Y, int *kind, int k, int d, int &fail) {
        const int kl = k - d;
        const int kE = kind[k], kt = kind[kl];
        __syncwarp(mask);
        T *Yk = Y + (size_t)k * L::SIZE, *Yl = Y + (size_t)kl * L::SIZE;
        wcopy<T, L::SIZE, WS>(s.e1, Yl, lane);
        wcopy<T, L::SIZE, WS>(s.e2, Yk, lane);
        __syncwarp(mask);
        wcopy<T, L::SIZE, WS>(Yl, s.e2, lane);
        if (kE == SLOT_IDENT) {
            wcopy<T, L::SIZE, WS>(Yk, s.e1, lane);
            if (lane == 0) { kind[kl] = kE; kind[k] = kt; }
        } else if (kt == SLOT_IDENT) {
            if (lane == 0) { kind[kl] = kE; kind[k] = kE; }
        } else {
            T Po[NX], po;
            if (!combine_cheap<T, NX, WS>(s, mask, lane, Po, po)) fail = min(fail, 1);
            SB::store_suffix_rows(Yk, Po, po, lane);
            if (lane == 0) { kind[kl] = kE; kind[k] = SLOT_ANCHOR; }
        }
        __syncwarp(mask);
    }
    // phase 3: chunk j < J-1 folded right-to-left from its exclusive suffix T_j = Y[J-1-j]
    static __device__ void phase3(CombineSmem<T, NX> &s, unsigned mask, int lane, const T *E, const T *Y, T *Pp, int j,
                                  int chunk, int J, int L2, int &fail) {
        const int lo = j * chunk, hi = min(lo + chunk, L2);
        wcopy<T, L::SIZE, WS>(s.e2, Y + (size_t)(J - 1 - j) * L::SIZE, lane);
        __syncwarp(mask);
        for (int i = hi - 1; i >= lo; --i) {
            wcopy<T, L::SIZE, WS>(s.e1, E + (size_t)i * L::SIZE, lane);
            __syncwarp(mask);
            T Po[NX], po;
            if (!combine_cheap<T, NX, WS>(s, mask, lane, Po, po)) fail = min(fail, i + 1);
            if (lane < NX) {
                st_row<T, NX, true>(s.e2 + L::P + lane * NX, Po);
                s.e2[L::p + lane] = po;
            }
            SB::out_Pp(Pp + (size_t)i * TP, Po, po, lane);
            __syncwarp(mask);
        }
    }
};

// CTA = IPB instances x W workers (all instances of a CTA run the same level schedule).
template <typename T, int NX>
__global__ void __launch_bounds__(256) k_scan_bwd(int B, int N, int chunk, int J, int Pv, int W, int IPB, LqWork<T> ws) {
    using U = BwdUnits<T, NX>;
    using L = VE<NX>;
    constexpr int WS = U::WS;
    constexpr int TP = TE<NX>::SIZE;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int WI = W * WS, ib = threadIdx.x / WI, w = (threadIdx.x % WI) / WS, lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    CombineSmem<T, NX> &s = reinterpret_cast<CombineSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    int *kind = reinterpret_cast<int *>(smraw + IPB * W * sizeof(CombineSmem<T, NX>)) + ib * Pv;
    const int b = blockIdx.x * IPB + ib, L2 = N + 2;
    const bool active = b < B;
    const int wv = active ? w : (INT_MAX / 2);  // inactive instances skip all work but reach every barrier
    const int b_ = active ? b : 0;
    const T *E = ws.elems + (size_t)b_ * L2 * L::SIZE;
    T *Y = ws.vslots + (size_t)b_ * Pv * L::SIZE;
    T *Pp = ws.Pp + (size_t)b_ * L2 * TP;
    int fail = INT_MAX;
    for (int j = wv; j < J; j += W) U::phase1(s, mask, lane, E, Y, kind, Pp, j, chunk, J, L2, fail);
    for (int t = J + (threadIdx.x % WI); t < Pv; t += WI) kind[t] = SLOT_IDENT;
    __syncthreads();
    if (J > 1) {
        for (int d = 1; d < Pv; d <<= 1) {
            const int np = Pv / (2 * d);
            for (int q = wv; q < np; q += W) U::up(s, mask, lane, Y, kind, 2 * d * (q + 1) - 1, d, fail);
            __syncthreads();
        }
        if (threadIdx.x % WI == 0) kind[Pv - 1] = SLOT_IDENT;
        __syncthreads();
        for (int d = Pv / 2; d >= 1; d >>= 1) {
            const int np = Pv / (2 * d);
            for (int q = wv; q < np; q += W) U::down(s, mask, lane, Y, kind, 2 * d * (q + 1) - 1, d, fail);
            __syncthreads();
        }
        for (int j = wv; j < J - 1; j += W) U::phase3(s, mask, lane, E, Y, Pp, j, chunk, J, L2, fail);
    }
    if (active && fail != INT_MAX && lane == 0) atomicMin(ws.fail + b, (1 << 24) | fail);
}

// Grid-wide variant for the latency regime (few instances): the units of every level are spread
// over all CTAs of a cooperative launch and the levels are separated by grid-wide barriers, so the
// span is 2 ceil(log2 J) combine latencies regardless of N (Eq. 8).  Slot kinds live in
// global memory (`kinds`: [B][Pv]).
template <typename T, int NX>
__global__ void __launch_bounds__(128) k_scan_bwd_grid(int B, int N, int chunk, int J, int Pv, LqWork<T> ws, int *kinds) {
    using U = BwdUnits<T, NX>;
    using L = VE<NX>;
    constexpr int WS = U::WS;
    constexpr int TP = TE<NX>::SIZE;
    extern __shared__ __align__(16) unsigned char smraw[];
    cg::grid_group grid = cg::this_grid();
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    CombineSmem<T, NX> &s = reinterpret_cast<CombineSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    const int wpb = blockDim.x / WS;
    const long gw = (long)blockIdx.x * wpb + threadIdx.x / WS, GW = (long)gridDim.x * wpb;
    const int L2 = N + 2;
    auto inst = [&](int b, const T *&E, T *&Y, T *&Pp, int *&kind) {
        E = ws.elems + (size_t)b * L2 * L::SIZE;
        Y = ws.vslots + (size_t)b * Pv * L::SIZE;
        Pp = ws.Pp + (size_t)b * L2 * TP;
        kind = kinds + (size_t)b * Pv;
    };
    auto report = [&](int b, int fail) {
        if (fail != INT_MAX && lane == 0) atomicMin(ws.fail + b, (1 << 24) | fail);
    };
    const T *E; T *Y; T *Pp; int *kind;
    for (long u = gw; u < (long)B * J; u += GW) {
        const int b = (int)(u / J), j = (int)(u % J);
        inst(b, E, Y, Pp, kind);
        int fail = INT_MAX;
        U::phase1(s, mask, lane, E, Y, kind, Pp, j, chunk, J, L2, fail);
        report(b, fail);
    }
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < (long)B * Pv; t += (long)gridDim.x * blockDim.x)
        if ((int)(t % Pv) >= J) kinds[t] = SLOT_IDENT;
    if (J == 1) return;
    grid.sync();
    for (int d = 1; d < Pv; d <<= 1) {
        const int np = Pv / (2 * d);
        for (long u = gw; u < (long)B * np; u += GW) {
            const int b = (int)(u / np), q = (int)(u % np);
            inst(b, E, Y, Pp, kind);
            int fail = INT_MAX;
            U::up(s, mask, lane, Y, kind, 2 * d * (q + 1) - 1, d, fail);
            report(b, fail);
        }
        grid.sync();
    }
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < B; t += (long)gridDim.x * blockDim.x)
        kinds[t * Pv + Pv - 1] = SLOT_IDENT;
    grid.sync();
    for (int d = Pv / 2; d >= 1; d >>= 1) {
        const int np = Pv / (2 * d);
        for (long u = gw; u < (long)B * np; u += GW) {
            const int b = (int)(u / np), q = (int)(u % np);
            inst(b, E, Y, Pp, kind);
            int fail = INT_MAX;
            U::down(s, mask, lane, Y, kind, 2 * d * (q + 1) - 1, d, fail);
            report(b, fail);
        }
        grid.sync();
    }
    for (long u = gw; u < (long)B * (J - 1); u += GW) {
        const int b = (int)(u / (J - 1)), j = (int)(u % (J - 1));
        inst(b, E, Y, Pp, kind);
        int fail = INT_MAX;
        U::phase3(s, mask, lane, E, Y, Pp, j, chunk, J, L2, fail);
        report(b, fail);
    }
}

// Full combination rule with the two half-warps of one warp cooperating (latency regime, D9): both
// halves form M = I + C1 P2 and run the same pivoted elimination (identical pivots); half 0 solves
// for [A1 | b1 - C1 p2] -> X, z and forms A = A2 X, b = A2 z + b2, V = P2 X, then P = A1^T V + P1,
// p = X^T w + p1; half 1 solves for C1 -> Y and forms C = A2 Y A2^T + C2 (same arithmetic per entry
// as combine_full, the critical path is one elimination with 13 instead of 25 right-hand sides and
// three instead of six products).  The result element is stored to dst (global).  Requires the
// whole warp converged; `s` is shared by the two halves.
template <typename T, int NX>
__device__ __forceinline__ bool combine_full_split(CombineSmem<T, NX> &s, T *dst) {
    using L = VE<NX>;
    static_assert(worker_width(NX) == 16, "half-warp workers");
    constexpr int WS = 16;
    const int lane = threadIdx.x & 15, half = (threadIdx.x >> 4) & 1;
    const unsigned mask = worker_mask<WS>();
    const int r = lane < NX ? lane : 0;
    T c1[NX];
    ld_row<T, NX, true>(c1, s.e1 + L::C + r * NX);
    T M[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) M[j] = (j == r) ? T(1) : T(0);
    row_mat<T, NX, NX, NX>(M, c1, s.e2 + L::P);
    bool ok;
    int pr;
    if (half == 0) {
        T rhs[NX + 1];
        ld_row<T, NX, true>(*reinterpret_cast<T(*)[NX]>(rhs), s.e1 + L::A + r * NX);
        rhs[NX] = s.e1[L::b + r] - row_dot<T, NX>(c1, s.e2 + L::p, T(0));
        ok = gauss_jordan<T, WS, NX, NX + 1, true>(mask, M, rhs, lane, NX, pr);
        if (pr >= 0) {
            st_row<T, NX, true>(s.X + pr * NX, *reinterpret_cast<T(*)[NX]>(rhs));
            s.z[pr] = rhs[NX];
        }
    } else {
        T rhs[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) rhs[j] = c1[j];
        ok = gauss_jordan<T, WS, NX, NX, true>(mask, M, rhs, lane, NX, pr);
        if (pr >= 0) st_row<T, NX, true>(s.Y + pr * NX, rhs);
    }
    __syncwarp();
    T a2[NX];
    ld_row<T, NX, true>(a2, s.e2 + L::A + r * NX);
    if (half == 0) {
        T Ao[NX];
        zero(Ao);
        row_mat<T, NX, NX, NX>(Ao, a2, s.X);
        const T bo = row_dot<T, NX>(a2, s.z, s.e2[L::b + r]);
        T p2[NX];
        ld_row<T, NX, true>(p2, s.e2 + L::P + r * NX);
        T V[NX];
        zero(V);
        row_mat<T, NX, NX, NX>(V, p2, s.X);
        const T wr = row_dot<T, NX>(p2, s.e1 + L::b, s.e2[L::p + r]);
        if (lane < NX) {
            st_row<T, NX, true>(s.V + r * NX, V);
            s.w[r] = wr;
            st_row<T, NX, true>(dst + L::A + r * NX, Ao);
            dst[L::b + r] = bo;
        }
        __syncwarp(mask);
        T a1c[NX], Po[NX];
        ld_col<T, NX>(a1c, s.e1 + L::A + r, NX);
        ld_row<T, NX, true>(Po, s.e1 + L::P + r * NX);
        row_mat<T, NX, NX, NX>(Po, a1c, s.V);
        T xc[NX];
        ld_col<T, NX>(xc, s.X + r, NX);
        const T po = row_dot<T, NX>(xc, s.w, s.e1[L::p + r]);
        __syncwarp(mask);
        symmetrize_rows<T, NX>(Po, s.V, mask, lane);
        if (lane < NX) {
            st_row<T, NX, true>(dst + L::P + r * NX, Po);
            dst[L::p + r] = po;
        }
    } else {
        T W[NX];
        zero(W);
        row_mat<T, NX, NX, NX>(W, a2, s.Y);
        T Co[NX];
        ld_row<T, NX, true>(Co, s.e2 + L::C + r * NX);
        row_matT<T, NX, NX, NX>(Co, W, s.e2 + L::A);
        __syncwarp(mask);
        symmetrize_rows<T, NX>(Co, s.Y, mask, lane);
        if (lane < NX) st_row<T, NX, true>(dst + L::C + r * NX, Co);
    }
    __syncwarp();
    return ok;
}

// Kogge-Stone reverse scan with one warp per combine (half-warp split of the full rule above, the
// cheap rule on half 0).  Same schedule and results as k_scan_bwd_ks.
template <typename T, int NX>
__global__ void __launch_bounds__(128) k_scan_bwd_ks2(int B, int N, int Pv, LqWork<T> ws) {
    using SB = ScanBwd<T, NX>;
    using L = VE<NX>;
    constexpr int TP = TE<NX>::SIZE;
    extern __shared__ __align__(16) unsigned char smraw[];
    cg::grid_group grid = cg::this_grid();
    const int wl = threadIdx.x & 31, lane = threadIdx.x & 15, half = (threadIdx.x >> 4) & 1;
    const unsigned hmask = worker_mask<16>();
    CombineSmem<T, NX> &s = reinterpret_cast<CombineSmem<T, NX> *>(smraw)[threadIdx.x / 32];
    const int wpb = blockDim.x / 32;
    const long gw = (long)blockIdx.x * wpb + threadIdx.x / 32, GW = (long)gridDim.x * wpb;
    const int L2 = N + 2;
    auto buf = [&](int k, int b, int i) -> T * {
        return k == 0 ? ws.elems + ((size_t)b * L2 + i) * L::SIZE : ws.vslots + ((size_t)b * Pv + i) * L::SIZE;
    };
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < (long)B * TP; t += (long)gridDim.x * blockDim.x) {
        const int b = (int)(t / TP), k = (int)(t % TP);
        const T *e = buf(0, b, L2 - 1);
        ws.Pp[((size_t)b * L2 + L2 - 1) * TP + k] = k < NX * NX ? e[L::P + k] : e[L::p + (k - NX * NX)];
    }
    int cur = 0;
    for (int d = 1; d < L2; d <<= 1) {
        grid.sync();
        for (long u = gw; u < (long)B * L2; u += GW) {
            const int b = (int)(u / L2), i = (int)(u % L2);
            if (i + d >= L2) continue;
            bool ok = true;
            wcopy<T, L::SIZE, 32>(s.e1, buf(cur, b, i), wl);
            if (i + 2 * d >= L2) {
                const T *Pr = ws.Pp + ((size_t)b * L2 + i + d) * TP;
                for (int k = wl; k < TP; k += 32) {
                    if (k < NX * NX) s.e2[L::P + k] = Pr[k];
                    else s.e2[L::p + (k - NX * NX)] = Pr[k];
                }
                __syncwarp();
                if (half == 0) {
                    T Po[NX], po;
                    ok = combine_cheap<T, NX, 16>(s, hmask, lane, Po, po);
                    SB::out_Pp(ws.Pp + ((size_t)b * L2 + i) * TP, Po, po, lane);
                }
            } else {
                wcopy<T, L::SIZE, 32>(s.e2, buf(cur, b, i + d), wl);
                __syncwarp();
                ok = combine_full_split<T, NX>(s, buf(cur ^ 1, b, i));
            }
            if (!ok && wl == 0) atomicMin(ws.fail + b, (1 << 24) | (i + 1));
            __syncwarp();
        }
        cur ^= 1;
    }
}

// Depth-optimal (Kogge-Stone) reverse scan for the latency regime (leaf chunk 1, few instances).
// Level d (d = 1, 2, 4, ...): every incomplete s_i becomes s_i (x) s_{i+d}.  At the start of level d,
// s_j covers stages [j, j + d) and is complete (the suffix through the terminal, R5) iff j + d >= L;
// a complete right operand is a suffix, so the cheap rule applies and the result is complete too.
// ceil(log2 L) dependent levels (6 at N = 50, 10 at N = 1000) instead of the Blelloch tree's
// 2 ceil(log2 L) + 1, for L log L combines instead of 2L -- chosen when a level fits in one wave of
// workers (D9).  Incomplete elements ping-pong between ws.elems (level-0 input) and
// ws.vslots (per-instance stride Pv >= L); a completed suffix lives only in ws.Pp as (P_i, p_i),
// which is all the cheap rule reads of its right operand.
template <typename T, int NX>
__global__ void __launch_bounds__(128) k_scan_bwd_ks(int B, int N, int Pv, LqWork<T> ws) {
    using SB = ScanBwd<T, NX>;
    using L = VE<NX>;
    constexpr int WS = worker_width(NX);
    constexpr int TP = TE<NX>::SIZE;
    extern __shared__ __align__(16) unsigned char smraw[];
    cg::grid_group grid = cg::this_grid();
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    CombineSmem<T, NX> &s = reinterpret_cast<CombineSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    const int wpb = blockDim.x / WS;
    const long gw = (long)blockIdx.x * wpb + threadIdx.x / WS, GW = (long)gridDim.x * wpb;
    const int L2 = N + 2;
    auto buf = [&](int k, int b, int i) -> T * {
        return k == 0 ? ws.elems + ((size_t)b * L2 + i) * L::SIZE : ws.vslots + ((size_t)b * Pv + i) * L::SIZE;
    };
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < (long)B * TP; t += (long)gridDim.x * blockDim.x) {
        const int b = (int)(t / TP), k = (int)(t % TP);   // s_{L-1} = e_{L-1} (terminal, Eq. 13)
        const T *e = buf(0, b, L2 - 1);
        ws.Pp[((size_t)b * L2 + L2 - 1) * TP + k] = k < NX * NX ? e[L::P + k] : e[L::p + (k - NX * NX)];
    }
    int cur = 0;
    for (int d = 1; d < L2; d <<= 1) {
        grid.sync();
        for (long u = gw; u < (long)B * L2; u += GW) {
            const int b = (int)(u / L2), i = (int)(u % L2);
            if (i + d >= L2) continue;  // s_i already complete
            int fail = INT_MAX;
            wcopy<T, L::SIZE, WS>(s.e1, buf(cur, b, i), lane);
            if (i + 2 * d >= L2) {  // right operand s_{i+d} complete: suffix (P, p) only
                const T *Pr = ws.Pp + ((size_t)b * L2 + i + d) * TP;
                for (int k = lane; k < TP; k += WS) {
                    if (k < NX * NX) s.e2[L::P + k] = Pr[k];
                    else s.e2[L::p + (k - NX * NX)] = Pr[k];
                }
                __syncwarp(mask);
                T Po[NX], po;
                if (!combine_cheap<T, NX, WS>(s, mask, lane, Po, po)) fail = i + 1;
                SB::out_Pp(ws.Pp + ((size_t)b * L2 + i) * TP, Po, po, lane);
            } else {
                wcopy<T, L::SIZE, WS>(s.e2, buf(cur, b, i + d), lane);
                __syncwarp(mask);
                T Ao[NX], Co[NX], Po[NX], bo, po;
                if (!combine_full<T, NX, WS>(s, mask, lane, Ao, Co, Po, bo, po)) fail = i + 1;
                SB::store_elem_rows(buf(cur ^ 1, b, i), Ao, Co, Po, bo, po, lane);
            }
            if (fail != INT_MAX && lane == 0) atomicMin(ws.fail + b, (1 << 24) | fail);
            __syncwarp(mask);
        }
        cur ^= 1;
    }
}

// ---------------------------------------------------------------------- policy (Eq. 5 rows)
// Per stage i (one worker):  PB = P_{i+1} B,  g = p_{i+1} + P_{i+1} b,
//   G = R + B^T PB,  H = S + PB^T A,  h = B^T g + r,  K = -G^-1 H,  k = -G^-1 h  (GJ, SPD),
//   Abar = A + B K,  bbar = B k + b   (Eq. 14).
template <typename T, int NX, int NU, bool EX>
__global__ void __launch_bounds__(128) k_policy(LqArgs<T> qp, int B, int N, int n, int m, LqWork<T> ws, LqOut<T> out) {
    constexpr int WS = worker_width(NX > NU ? NX : NU);
    constexpr int SMW = NX * NU + NX * NX + NX * NU + NU * NX + round_up4(NU) + NX + NX;  // B, A, PB, K, k, c, g
    using KL = KE<NX, NU>;
    constexpr int TP = TE<NX>::SIZE;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int wloc = threadIdx.x / WS;
    const long gw = (long)blockIdx.x * (blockDim.x / WS) + wloc;
    if (gw >= (long)B * (N + 1)) return;
    const int b = (int)(gw / (N + 1)), i = (int)(gw % (N + 1));
    T *sm = reinterpret_cast<T *>(smraw) + wloc * SMW;
    T *sB = sm, *sA = sB + NX * NU, *sPB = sA + NX * NX, *sK = sPB + NX * NU, *sk = sK + NU * NX;
    T *sc = sk + round_up4(NU), *sg = sc + NX;
    const size_t st = (size_t)b * (N + 1) + i;
    const int r = lane < NX ? lane : 0;
    const bool vr = EX || r < n;
    T brow[NU], arow[NX];
    if (vr) {
        ld_row<T, NU, EX>(brow, qp.Bm + st * n * m + r * m, m);
        ld_row<T, NX, EX>(arow, qp.A + st * n * n + r * n, n);
    } else {
        zero(brow);
        zero(arow);
    }
    const T cr = vr ? qp.c[st * n + r] : T(0);
    if (lane < NX) {
        st_row<T, NU, true>(sB + r * NU, brow);
        st_row<T, NX, true>(sA + r * NX, arow);
        sc[r] = cr;
    }
    __syncwarp(mask);
    const T *Pn = ws.Pp + ((size_t)b * (N + 2) + i + 1) * TP;
    {
        T prow[NX], pb[NU];
        ld_row<T, NX, true>(prow, Pn + r * NX);
        zero(pb);
        row_mat<T, NX, NU, NU>(pb, prow, sB);
        const T g = row_dot<T, NX>(prow, sc, Pn[NX * NX + r]);
        if (lane < NX) { st_row<T, NU, true>(sPB + r * NU, pb); sg[r] = g; }
    }
    __syncwarp(mask);
    {
        const int ru = lane < NU ? lane : 0;
        const bool vu = EX || ru < m;
        T G[NU], rhs[NX + 1];
        if (vu) {
            ld_row<T, NU, EX>(G, qp.R + st * m * m + ru * m, m);
            if (qp.S != nullptr) ld_row<T, NX, EX>(*reinterpret_cast<T(*)[NX]>(rhs), qp.S + st * m * n + ru * n, n);
            else zero(*reinterpret_cast<T(*)[NX]>(rhs));   // S = 0 (SRBD Gauss-Newton cost)
            rhs[NX] = qp.r[st * m + ru];
        } else {
#pragma unroll
            for (int j = 0; j < NU; ++j) G[j] = (j == ru) ? T(1) : T(0);
#pragma unroll
            for (int j = 0; j <= NX; ++j) rhs[j] = T(0);
        }
        T bcol[NX], pbcol[NX];
        ld_col<T, NX>(bcol, sB + ru, NU);
        ld_col<T, NX>(pbcol, sPB + ru, NU);
        row_mat<T, NX, NU, NU>(G, bcol, sPB);
        row_mat<T, NX, NX, NX>(*reinterpret_cast<T(*)[NX]>(rhs), pbcol, sA);
        rhs[NX] = row_dot<T, NX>(bcol, sg, rhs[NX]);
        int pr;
        const bool ok = gauss_jordan<T, WS, NU, NX + 1, false>(mask, G, rhs, lane, NU, pr);
        if (!ok && lane == 0) atomicMin(ws.fail + b, (2 << 24) | (i + 1));
        if (pr >= 0) {
            T kr[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) kr[j] = -rhs[j];
            st_row<T, NX, true>(sK + pr * NX, kr);
            sk[pr] = -rhs[NX];
            T *Kw = ws.Kk + st * KL::SIZE;
            st_row<T, NX, true>(Kw + KL::K + pr * NX, kr);
            Kw[KL::k + pr] = -rhs[NX];
            if (out.K != nullptr && (EX || pr < m)) st_row<T, NX, EX>(out.K + st * m * n + pr * n, kr, n);
            if (out.k != nullptr && (EX || pr < m)) out.k[st * m + pr] = -rhs[NX];
        }
    }
    __syncwarp(mask);
    T abar[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) abar[j] = arow[j];
    row_mat<T, NU, NX, NX>(abar, brow, sK);
    const T bb = row_dot<T, NU>(brow, sk, cr);
    if (lane < NX) {
        T *te = ws.tel + st * TP;
        st_row<T, NX, true>(te + r * NX, abar);
        te[NX * NX + r] = bb;
    }
}

// ------------------------------------------------------------ forward scan (Eq. 14-15, R6)
// Elements a_i = (Abar_i, bbar_i), i = 0..N; a_0 is anchored at dx_0 (Abar_{0,1} = 0,
// bbar_{0,1} = Abar_0 dx_0 + bbar_0).  Composition (a then b) = (Abar_b Abar_a, Abar_b bbar_a + bbar_b).
// Prefix a_0 (+) ... (+) a_i = (0, dx_{i+1}).  Same chunked Blelloch structure as k_scan_bwd.
template <typename T, int NX>
struct FwdSmem {
    T t1[TE<NX>::SIZE];
    T t2[TE<NX>::SIZE];
};

template <typename T, int NX>
struct FwdUnits {
    using TL = TE<NX>;
    static constexpr int WS = worker_width(NX);
    // dx_{i+1} = Abar_i dx_i + bbar_i for i in [lo, hi), x in s.t2[TL::b..]; writes dx (padded
    // workspace X and the user's Xo with n columns)
    static __device__ void fold(FwdSmem<T, NX> &s, unsigned mask, int lane, const T *E, T *X, T *Xo, int n, int lo, int hi) {
        const int r = lane < NX ? lane : 0;
        for (int i = lo; i < hi; ++i) {
            T arow[NX];
            ld_row<T, NX, true>(arow, E + (size_t)i * TL::SIZE + r * NX);
            const T v = row_dot<T, NX>(arow, s.t2 + TL::b, E[(size_t)i * TL::SIZE + TL::b + r]);
            __syncwarp(mask);
            if (lane < NX) {
                s.t2[TL::b + r] = v;
                X[(i + 1) * NX + r] = v;
                if (n == NX || r < n) Xo[(size_t)(i + 1) * n + r] = v;
            }
            __syncwarp(mask);
        }
    }
    static __device__ void phase1(FwdSmem<T, NX> &s, unsigned mask, int lane, const T *E, T *Y, int *kind, T *X, T *Xo,
                                  const T *dx0b, int n, int j, int chunk, int J, int Lf) {
        const int r = lane < NX ? lane : 0;
        const int lo = j * chunk, hi = min(lo + chunk, Lf);
        if (j == 0) {
            const T x0 = (n == NX || r < n) ? dx0b[r] : T(0);
            if (lane < NX) {
                s.t2[TL::b + r] = x0;
                X[r] = x0;
                if (n == NX || r < n) Xo[r] = x0;
            }
            __syncwarp(mask);
            fold(s, mask, lane, E, X, Xo, n, lo, hi);
            if (J > 1 && lane < NX) Y[TL::b + r] = s.t2[TL::b + r];
            if (lane == 0 && J > 1) kind[0] = SLOT_ANCHOR;
        } else {
            wcopy<T, TL::SIZE, WS>(s.t2, E + (size_t)lo * TL::SIZE, lane);
            __syncwarp(mask);
            for (int i = lo + 1; i < hi; ++i) {
                T arow[NX], ao[NX];
                ld_row<T, NX, true>(arow, E + (size_t)i * TL::SIZE + r * NX);
                zero(ao);
                row_mat<T, NX, NX, NX>(ao, arow, s.t2 + TL::A);
                const T bo = row_dot<T, NX>(arow, s.t2 + TL::b, E[(size_t)i * TL::SIZE + TL::b + r]);
                __syncwarp(mask);
                if (lane < NX) { st_row<T, NX, true>(s.t2 + TL::A + r * NX, ao); s.t2[TL::b + r] = bo; }
                __syncwarp(mask);
            }
            wcopy<T, TL::SIZE, WS>(Y + (size_t)j * TL::SIZE, s.t2, lane);
            if (lane == 0) kind[j] = SLOT_GENERAL;
        }
        __syncwarp(mask);
    }
    // up-sweep node k: Y[k] = Y[k-d] (+) Y[k]  (apply Y[k-d] first)
    static __device__ void up(FwdSmem<T, NX> &s, unsigned mask, int lane, T *Y, int *kind, int k, int d) {
        const int r = lane < NX ? lane : 0;
        const int kl = k - d;
        const int kk = kind[k], kp = kind[kl];
        __syncwarp(mask);
        T *Yk = Y + (size_t)k * TL::SIZE, *Yl = Y + (size_t)kl * TL::SIZE;
        if (kp == SLOT_IDENT) {
        } else if (kk == SLOT_IDENT) {
            wcopy<T, TL::SIZE, WS>(Yk, Yl, lane);
            if (lane == 0) kind[k] = kp;
        } else {
            wcopy<T, TL::SIZE, WS>(s.t1, Yl, lane);
            wcopy<T, TL::SIZE, WS>(s.t2, Yk, lane);
            __syncwarp(mask);
            T arow[NX];
            ld_row<T, NX, true>(arow, s.t2 + TL::A + r * NX);
            const T bo = row_dot<T, NX>(arow, s.t1 + TL::b, s.t2[TL::b + r]);
            if (kp == SLOT_ANCHOR) {
                if (lane < NX) Yk[TL::b + r] = bo;
                if (lane == 0) kind[k] = SLOT_ANCHOR;
            } else {
                T ao[NX];
                zero(ao);
                row_mat<T, NX, NX, NX>(ao, arow, s.t1 + TL::A);
                if (lane < NX) { st_row<T, NX, true>(Yk + TL::A + r * NX, ao); Yk[TL::b + r] = bo; }
            }
        }
        __syncwarp(mask);
    }
    // down-sweep node k: t = Y[k-d]; Y[k-d] = Y[k]; Y[k] = Y[k] (+) t  (prefix first, then t)
    static __device__ void down(FwdSmem<T, NX> &s, unsigned mask, int lane, T *Y, int *kind, int k, int d) {
        const int r = lane < NX ? lane : 0;
        const int kl = k - d;
        const int kE = kind[k], kt = kind[kl];
        __syncwarp(mask);
        T *Yk = Y + (size_t)k * TL::SIZE, *Yl = Y + (size_t)kl * TL::SIZE;
        wcopy<T, TL::SIZE, WS>(s.t1, Yl, lane);
        wcopy<T, TL::SIZE, WS>(s.t2, Yk, lane);
        __syncwarp(mask);
        wcopy<T, TL::SIZE, WS>(Yl, s.t2, lane);
        if (kE == SLOT_IDENT) {
            wcopy<T, TL::SIZE, WS>(Yk, s.t1, lane);
            if (lane == 0) { kind[kl] = kE; kind[k] = kt; }
        } else if (kt == SLOT_IDENT) {
            if (lane == 0) { kind[kl] = kE; kind[k] = kE; }
        } else {
            T arow[NX];
            ld_row<T, NX, true>(arow, s.t1 + TL::A + r * NX);
            const T bo = row_dot<T, NX>(arow, s.t2 + TL::b, s.t1[TL::b + r]);
            if (lane < NX) Yk[TL::b + r] = bo;
            if (lane == 0) { kind[kl] = kE; kind[k] = SLOT_ANCHOR; }
        }
        __syncwarp(mask);
    }
};

template <typename T, int NX>
__global__ void __launch_bounds__(256) k_scan_fwd(const T *dx0, int B, int N, int n, int chunk, int J, int Pf, int W,
                                                  int IPB, LqWork<T> ws, T *dx_out) {
    using U = FwdUnits<T, NX>;
    using TL = TE<NX>;
    constexpr int WS = U::WS;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int WI = W * WS, ib = threadIdx.x / WI, w = (threadIdx.x % WI) / WS, lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    FwdSmem<T, NX> &s = reinterpret_cast<FwdSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    int *kind = reinterpret_cast<int *>(smraw + IPB * W * sizeof(FwdSmem<T, NX>)) + ib * Pf;
    const int b = blockIdx.x * IPB + ib, Lf = N + 1;
    const bool active = b < B;
    const int b_ = active ? b : 0;
    const T *E = ws.tel + (size_t)b_ * Lf * TL::SIZE;
    T *Y = ws.tslots + (size_t)b_ * Pf * TL::SIZE;
    T *X = ws.dxw + (size_t)b_ * (N + 2) * NX;
    T *Xo = dx_out + (size_t)b_ * (N + 2) * n;
    const int wv = active ? w : (INT_MAX / 2);  // inactive instances skip all work but reach every barrier
    for (int j = wv; j < J; j += W) U::phase1(s, mask, lane, E, Y, kind, X, Xo, dx0 + (size_t)b_ * n, n, j, chunk, J, Lf);
    for (int t = J + (threadIdx.x % WI); t < Pf; t += WI) kind[t] = SLOT_IDENT;
    __syncthreads();
    if (J > 1) {
        for (int d = 1; d < Pf; d <<= 1) {
            const int np = Pf / (2 * d);
            for (int q = wv; q < np; q += W) U::up(s, mask, lane, Y, kind, 2 * d * (q + 1) - 1, d);
            __syncthreads();
        }
        if (threadIdx.x % WI == 0) kind[Pf - 1] = SLOT_IDENT;
        __syncthreads();
        for (int d = Pf / 2; d >= 1; d >>= 1) {
            const int np = Pf / (2 * d);
            for (int q = wv; q < np; q += W) U::down(s, mask, lane, Y, kind, 2 * d * (q + 1) - 1, d);
            __syncthreads();
        }
        for (int j = wv > 0 ? wv : W; j < J; j += W) {   // phase 3: chunks j >= 1 from their prefix
            const int lo = j * chunk, hi = min(lo + chunk, Lf);
            const int r = lane < NX ? lane : 0;
            if (lane < NX) s.t2[TL::b + r] = Y[(size_t)j * TL::SIZE + TL::b + r];
            __syncwarp(mask);
            U::fold(s, mask, lane, E, X, Xo, n, lo, hi);
        }
    }
}

// Grid-wide forward scan (cooperative launch), companion of k_scan_bwd_grid.
template <typename T, int NX>
__global__ void __launch_bounds__(128) k_scan_fwd_grid(const T *dx0, int B, int N, int n, int chunk, int J, int Pf,
                                                       LqWork<T> ws, T *dx_out, int *kinds) {
    using U = FwdUnits<T, NX>;
    using TL = TE<NX>;
    constexpr int WS = U::WS;
    extern __shared__ __align__(16) unsigned char smraw[];
    cg::grid_group grid = cg::this_grid();
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    FwdSmem<T, NX> &s = reinterpret_cast<FwdSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    const int wpb = blockDim.x / WS;
    const long gw = (long)blockIdx.x * wpb + threadIdx.x / WS, GW = (long)gridDim.x * wpb;
    const int Lf = N + 1;
    auto E_ = [&](int b) { return ws.tel + (size_t)b * Lf * TL::SIZE; };
    auto Y_ = [&](int b) { return ws.tslots + (size_t)b * Pf * TL::SIZE; };
    auto X_ = [&](int b) { return ws.dxw + (size_t)b * (N + 2) * NX; };
    auto Xo_ = [&](int b) { return dx_out + (size_t)b * (N + 2) * n; };
    for (long u = gw; u < (long)B * J; u += GW) {
        const int b = (int)(u / J), j = (int)(u % J);
        U::phase1(s, mask, lane, E_(b), Y_(b), kinds + (size_t)b * Pf, X_(b), Xo_(b), dx0 + (size_t)b * n, n, j, chunk, J, Lf);
    }
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < (long)B * Pf; t += (long)gridDim.x * blockDim.x)
        if ((int)(t % Pf) >= J) kinds[t] = SLOT_IDENT;
    if (J == 1) return;
    grid.sync();
    for (int d = 1; d < Pf; d <<= 1) {
        const int np = Pf / (2 * d);
        for (long u = gw; u < (long)B * np; u += GW) {
            const int b = (int)(u / np), q = (int)(u % np);
            U::up(s, mask, lane, Y_(b), kinds + (size_t)b * Pf, 2 * d * (q + 1) - 1, d);
        }
        grid.sync();
    }
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < B; t += (long)gridDim.x * blockDim.x)
        kinds[t * Pf + Pf - 1] = SLOT_IDENT;
    grid.sync();
    for (int d = Pf / 2; d >= 1; d >>= 1) {
        const int np = Pf / (2 * d);
        for (long u = gw; u < (long)B * np; u += GW) {
            const int b = (int)(u / np), q = (int)(u % np);
            U::down(s, mask, lane, Y_(b), kinds + (size_t)b * Pf, 2 * d * (q + 1) - 1, d);
        }
        grid.sync();
    }
    for (long u = gw; u < (long)B * (J - 1); u += GW) {
        const int b = (int)(u / (J - 1)), j = 1 + (int)(u % (J - 1));
        const int lo = j * chunk, hi = min(lo + chunk, Lf);
        const int r = lane < NX ? lane : 0;
        if (lane < NX) s.t2[TL::b + r] = Y_(b)[(size_t)j * TL::SIZE + TL::b + r];
        __syncwarp(mask);
        U::fold(s, mask, lane, E_(b), X_(b), Xo_(b), n, lo, hi);
    }
}

// Depth-optimal (Kogge-Stone) forward scan, companion of k_scan_bwd_ks (D9).  t_j covers elements
// (j - d, j] at the start of level d and is complete -- anchored at dx_0, i.e. (0, dx_{j+1}) -- iff
// j < d.  Level d: every incomplete t_i (i >= d) becomes t_{i-d} then t_i; when t_{i-d} is complete
// the result is dx_{i+1} = Abar_(i) dx_{i-d+1} + bbar_(i), written to the padded workspace X and to
// the user's dx.  Incomplete composites ping-pong between ws.tel (level-0 input) and ws.tslots.
template <typename T, int NX>
__global__ void __launch_bounds__(128) k_scan_fwd_ks(const T *dx0, int B, int N, int n, int Pf, LqWork<T> ws, T *dx_out) {
    using TL = TE<NX>;
    constexpr int WS = worker_width(NX);
    extern __shared__ __align__(16) unsigned char smraw[];
    cg::grid_group grid = cg::this_grid();
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    FwdSmem<T, NX> &s = reinterpret_cast<FwdSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    const int wpb = blockDim.x / WS;
    const long gw = (long)blockIdx.x * wpb + threadIdx.x / WS, GW = (long)gridDim.x * wpb;
    const int Lf = N + 1, r = lane < NX ? lane : 0;
    const bool vr = lane < NX && (n == NX || r < n);
    auto buf = [&](int k, int b, int i) -> T * {
        return k == 0 ? ws.tel + ((size_t)b * Lf + i) * TL::SIZE : ws.tslots + ((size_t)b * Pf + i) * TL::SIZE;
    };
    for (long b = gw; b < B; b += GW) {  // anchor: dx_0, and t_0 = (0, dx_1 = Abar_0 dx_0 + bbar_0)
        T *X = ws.dxw + (size_t)b * (N + 2) * NX, *Xo = dx_out + (size_t)b * (N + 2) * n;
        const T x0 = vr ? dx0[(size_t)b * n + r] : T(0);
        if (lane < NX) { s.t2[TL::b + r] = x0; X[r] = x0; }
        if (vr) Xo[r] = x0;
        __syncwarp(mask);
        const T *E = buf(0, (int)b, 0);
        T arow[NX];
        ld_row<T, NX, true>(arow, E + r * NX);
        const T v = row_dot<T, NX>(arow, s.t2 + TL::b, E[TL::b + r]);
        if (lane < NX) X[NX + r] = v;
        if (vr) Xo[n + r] = v;
        __syncwarp(mask);
    }
    int cur = 0;
    for (int d = 1; d < Lf; d <<= 1) {
        grid.sync();
        for (long u = gw; u < (long)B * Lf; u += GW) {
            const int b = (int)(u / Lf), i = (int)(u % Lf);
            if (i < d) continue;  // t_i complete
            T *X = ws.dxw + (size_t)b * (N + 2) * NX;
            const T *Ei = buf(cur, b, i);
            T arow[NX];
            ld_row<T, NX, true>(arow, Ei + r * NX);
            if (i < 2 * d) {  // left operand complete: dx_{i+1}
                const T v = row_dot<T, NX>(arow, X + (size_t)(i - d + 1) * NX, Ei[TL::b + r]);
                if (lane < NX) X[(size_t)(i + 1) * NX + r] = v;
                if (vr) dx_out[((size_t)b * (N + 2) + i + 1) * n + r] = v;
            } else {
                wcopy<T, TL::SIZE, WS>(s.t1, buf(cur, b, i - d), lane);
                __syncwarp(mask);
                T ao[NX];
                zero(ao);
                row_mat<T, NX, NX, NX>(ao, arow, s.t1 + TL::A);
                const T bo = row_dot<T, NX>(arow, s.t1 + TL::b, Ei[TL::b + r]);
                T *D = buf(cur ^ 1, b, i);
                if (lane < NX) { st_row<T, NX, true>(D + TL::A + r * NX, ao); D[TL::b + r] = bo; }
            }
            __syncwarp(mask);
        }
        cur ^= 1;
    }
}

// ------------------------------------------------------------ tail: du (Eq. 6), dlam (Eq. 7)
template <typename T, int NX, int NU>
__global__ void k_tail(int B, int N, int n, int m, LqWork<T> ws, LqOut<T> out) {
    using KL = KE<NX, NU>;
    constexpr int TP = TE<NX>::SIZE;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long per = (long)(N + 1) * m + (long)(N + 2) * n;
    if (t >= (long)B * per) return;
    const int b = (int)(t / per);
    int rem = (int)(t % per);
    const T *x = ws.dxw + (size_t)b * (N + 2) * NX;
    T v;
    bool bad;
    if (rem < (N + 1) * m) {
        const int i = rem / m, a = rem % m;
        const T *K = ws.Kk + ((size_t)b * (N + 1) + i) * KL::SIZE;
        v = K[KL::k + a];
#pragma unroll
        for (int j = 0; j < NX; ++j) v = fma(K[KL::K + a * NX + j], x[i * NX + j], v);
        out.du[(size_t)b * (N + 1) * m + rem] = v;
        bad = !isfinite(v) || !isfinite(x[i * NX + (a < n ? a : 0)]);
    } else {
        rem -= (N + 1) * m;
        const int i = rem / n, a = rem % n;
        const T *Pp = ws.Pp + ((size_t)b * (N + 2) + i) * TP;
        v = Pp[NX * NX + a];
#pragma unroll
        for (int j = 0; j < NX; ++j) v = fma(Pp[a * NX + j], x[i * NX + j], v);
        out.dlam[(size_t)b * (N + 2) * n + rem] = v;
        bad = !isfinite(v) || !isfinite(x[i * NX + a]);
    }
    if (bad) ws.nonfin[b] = 1;
}

// info[b] = factorisation failure stage (k > 0), else -1 if a non-finite output, else 0.
// Failures are ranked by origin (R in element init < scan combine < G in the policy), then by
// stage: fail[b] = (origin << 24) | (stage + 1), min over all failures.
static __global__ void k_finalize_info(int B, const int32_t *fail, const int32_t *nonfin, const int32_t *pre,
                                       int32_t *info) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int v = fail[b] != kFailNone ? (fail[b] & 0xFFFFFF) : (nonfin[b] ? -1 : 0);
    if (pre != nullptr && pre[b] != 0) v = pre[b];
    info[b] = v;
}

// ------------------------------------------------------------ single-chunk reverse scan (J = 1)
// s_{N+1} = e_{N+1}, s_i = e_i (x) s_{i+1} by the cheap rule for i = N..0: the leaf_chunk >= N+2
// schedule of k_scan_bwd as a tight per-instance loop.  Two instances per warp, warp kept
// converged (a worker past the batch recomputes instance B-1 without storing); the next element is
// prefetched into shared memory with cp.async while the current combine runs; compact Gauss-Jordan
// keeps the loop body small.
template <typename T, int NX>
struct FoldChainSmem {
    T buf[2][VE<NX>::SIZE];
    T P[NX * NX], X[NX * NX], V[NX * NX];
    T p[NX], w[NX];
};

template <typename T, int NX, int MINB>
__global__ void __launch_bounds__(128, MINB) k_fold(int B, int N, LqWork<T> ws) {
    constexpr int WS = worker_width(NX);
    using L = VE<NX>;
    constexpr int TP = TE<NX>::SIZE;
    constexpr int NG = L::SIZE * sizeof(T) / 16;  // 16-byte granules per element
    extern __shared__ __align__(16) unsigned char smraw[];
    FoldChainSmem<T, NX> &s = reinterpret_cast<FoldChainSmem<T, NX> *>(smraw)[threadIdx.x / WS];
    const int lane = worker_lane<WS>();
    const int b_raw = blockIdx.x * (blockDim.x / WS) + threadIdx.x / WS;
    if (__all_sync(0xffffffffu, b_raw >= B)) return;
    const bool live = b_raw < B;
    const int b = live ? b_raw : B - 1;
    const int r = lane < NX ? lane : 0;
    const bool act = lane < NX;
    const T *E = ws.elems + (size_t)b * (N + 2) * L::SIZE;
    T *Pp = ws.Pp + (size_t)b * (N + 2) * TP;
    auto prefetch = [&](int i, int slot) {
        const char *src = reinterpret_cast<const char *>(E + (size_t)i * L::SIZE);
        char *dst = reinterpret_cast<char *>(s.buf[slot]);
        for (int g = lane; g < NG; g += WS) cp_async16(dst + 16 * g, src + 16 * g);
    };
    prefetch(N, 0);
    cp_async_commit();
    {  // s_{N+1} = e_{N+1}: only P~, p~ are nonzero (Eq. 13)
        T prow[NX];
        ld_row<T, NX, true>(prow, E + (size_t)(N + 1) * L::SIZE + L::P + r * NX);
        const T pr = E[(size_t)(N + 1) * L::SIZE + L::p + r];
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, prow);
            s.p[r] = pr;
            if (live) {
                st_row<T, NX, true>(Pp + (size_t)(N + 1) * TP + r * NX, prow);
                Pp[(size_t)(N + 1) * TP + NX * NX + r] = pr;
            }
        }
    }
    int fail = INT_MAX;
    for (int i = N; i >= 0; --i) {
        const int cur = (N - i) & 1;
        if (i > 0) prefetch(i - 1, cur ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const T *e1 = s.buf[cur];
        T prow[NX];
        ld_row<T, NX, true>(prow, s.P + r * NX);
        T M[NX];
        {
            T c1[NX];
            ld_row<T, NX, true>(c1, e1 + L::C + r * NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) M[j] = (j == r) ? T(1) : T(0);
            row_mat<T, NX, NX, NX>(M, c1, s.P);                      // M = I + C~_i P_{i+1}
        }
        const T wr = row_dot<T, NX>(prow, e1 + L::b, s.p[r]);        // w = p' + P' b~_i
        if (act) s.w[r] = wr;
        T rhs[NX];
        ld_row<T, NX, true>(rhs, e1 + L::A + r * NX);
        int pr;
        if (!gauss_jordan<T, WS, NX, NX, true, true>(0xffffffffu, M, rhs, lane, NX, pr)) fail = min(fail, i + 1);
        if (pr >= 0) st_row<T, NX, true>(s.X + pr * NX, rhs);       // X = M^-1 A~_i
        __syncwarp();
        {
            T V[NX];
            zero(V);
            row_mat<T, NX, NX, NX>(V, prow, s.X);                    // V = P' X
            if (act) st_row<T, NX, true>(s.V + r * NX, V);
        }
        T pn;
        {
            T xc[NX];
            ld_col<T, NX>(xc, s.X + r, NX);
            pn = row_dot<T, NX>(xc, s.w, e1[L::p + r]);              // p_i = X^T w + p~_i
        }
        __syncwarp();
        T Pn[NX];
        {
            T ac[NX];
            ld_col<T, NX>(ac, e1 + L::A + r, NX);
            ld_row<T, NX, true>(Pn, e1 + L::P + r * NX);
            row_mat<T, NX, NX, NX>(Pn, ac, s.V);                     // P_i = A~^T P' X + P~_i
        }
        __syncwarp();
        symmetrize_rows<T, NX>(Pn, s.X, 0xffffffffu, lane);
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, Pn);
            s.p[r] = pn;
            if (live) {
                st_row<T, NX, true>(Pp + (size_t)i * TP + r * NX, Pn);
                Pp[(size_t)i * TP + NX * NX + r] = pn;
            }
        }
        __syncwarp();
    }
    if (live && fail != INT_MAX && lane == 0) atomicMin(ws.fail + b, (1 << 24) | fail);
}

}  // namespace pdilqr
