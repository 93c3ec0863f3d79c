// srbd_fused.cuh -- fused SRBD step for the single-chunk schedule (leaf_chunk >= N+2): the
// reverse associative scan degenerates to a right-to-left fold of cheap combines, so the whole
// backward pass of one instance runs in one worker with every per-stage quantity on chip.
//
//   k_srbd_bwd_fold  for i = N .. 0 (one 16-lane worker per instance, lane r owns row r):
//       linearise stage i  ->  element e_i (Eq. 12, S = 0)  ->
//       policy K_i, k_i from P_{i+1}, p_{i+1} (Eq. 5 rows) and (Abar_i, bbar_i) (Eq. 14)  ->
//       s_i = e_i (x) s_{i+1} by the cheap combination rule (Eq. 11, readings R1-R2).
//     Writes (K_i, k_i), (Abar_i, bbar_i), (P_i, p_i) per stage; nothing else leaves the SM.
//   k_srbd_fwd_ls    one warp per instance: closed-loop rollout dx_{i+1} = Abar_i dx_i + bbar_i
//       (the forward scan of Eq. 15 with one chunk), du_i = K_i dx_i + k_i (Eq. 6),
//       dlam_i = P_i dx_i + p_i (Eq. 7), then the parallel filter line search over the alpha
//       grid (lanes over stages) and the in-place update (Eq. 16).
#pragma once

#include "srbd.cuh"

namespace pdilqr {

// SFU fast math in fp32 (line search only: evaluations whose rounding cannot change the LQ solve);
// accurate libm in fp64.
__device__ __forceinline__ void fast_sincos(float x, float *s, float *c) { __sincosf(x, s, c); }
__device__ __forceinline__ void fast_sincos(double x, double *s, double *c) { sincos(x, s, c); }
__device__ __forceinline__ float fast_log(float x) { return __logf(x); }
__device__ __forceinline__ double fast_log(double x) { return log(x); }

template <typename T>
struct LsWarps {  // k_srbd_fwd_ls block = LsWarps * 32 threads (static shared memory <= 48 KB)
    static constexpr int value = sizeof(T) == 8 ? 2 : 4;
};

template <typename T>
struct FoldSmem {
    T P[144], A[144], B[144], ZB[144], X[144], V[144], K[144];
    T p[12], c[12], g[12], bt[12], w[12], zr[12], k[12], pad[4];
    // per-stage inputs staged by cp.async one stage ahead (3 slots: stage i-1 lands while stages
    // i and i+1 are read): x, lam, xref, u, feet, uref (12 each), contact flags (4 bytes at IN_CON)
    static constexpr int IN_X = 0, IN_L = 12, IN_XR = 24, IN_U = 36, IN_F = 48, IN_UR = 60, IN_CON = 72, IN = 80;
    T in[3][IN];
};

// TPB threads per block (2 workers per warp); MINB * 128 / TPB blocks per SM keep the 128-register
// cap.  Small blocks balance the one-wave grid across the 148 SMs (B = 4096: 512 blocks of 128
// threads put 4 blocks on 68 SMs and 3 on 80; 1024 blocks of 64 threads put 7 or 6).
template <typename T, int MINB, int TPB = 64, bool LM = false>
__global__ void __launch_bounds__(TPB, MINB * 128 / TPB) k_srbd_bwd_fold(SrbdConst K, SrbdIter<T> it, int B, int N, LqWork<T> ws,
                                                             int32_t *info_out) {
    constexpr int WS = 16, NX = 12;
    constexpr int TP = TE<NX>::SIZE;
    using KL = KE<NX, NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    FoldSmem<T> &s = reinterpret_cast<FoldSmem<T> *>(smraw)[threadIdx.x / WS];
    const int lane = worker_lane<WS>();
    // The warp stays converged: both workers run the same schedule; a worker past the end of the
    // batch recomputes instance B-1 and stores nothing.  All warp collectives use the full mask.
    const unsigned mask = 0xffffffffu;
    const int b_raw = blockIdx.x * (blockDim.x / WS) + threadIdx.x / WS;
    if (__all_sync(0xffffffffu, b_raw >= B)) return;
    const bool live = b_raw < B;
    const int b = live ? b_raw : B - 1;
    const int r = lane < NX ? lane : 0;
    const bool act = lane < NX;
    const bool wr_g = act && live;  // global stores
    const T *xb = it.x + (size_t)b * (N + 2) * NX;
    const T *lb = it.lam + (size_t)b * (N + 2) * NX;
    const T *xrb = it.xref + (size_t)b * (N + 2) * NX;
    T *Pp = ws.Pp + (size_t)b * (N + 2) * TP;
    T *Kk = ws.Kk + (size_t)b * (N + 1) * KL::SIZE;
    T *Te = ws.tel + (size_t)b * (N + 1) * TP;
    const T dt = T(K.dt);
    bool bad = false;
    int fail = INT_MAX;
    // terminal element e_{N+1} = suffix s_{N+1}: P = W_N, p = W_N (x_{N+1} - xref) - lam_{N+1}  (Eq. 13)
    {
        const T xr = xb[(N + 1) * NX + r], lr = lb[(N + 1) * NX + r];
        T Prow[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) Prow[j] = (j == r) ? T(K.wxt[r]) : T(0);
        const T pr = T(K.wxt[r]) * (xr - xrb[(N + 1) * NX + r]) - lr;
        bad = bad || !isfinite(xr) || !isfinite(lr);
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, Prow);
            s.p[r] = pr;
        }
        if (wr_g) {
            st_row<T, NX, true>(Pp + (size_t)(N + 1) * TP + r * NX, Prow);
            Pp[(size_t)(N + 1) * TP + NX * NX + r] = pr;
        }
    }
    // stage inputs -> s.in[stage % 3] (cp.async, 16-byte chunks spread over the worker's lanes)
    using FS = FoldSmem<T>;
    constexpr int EPC = 16 / (int)sizeof(T), RCH = NX / EPC;  // elements / chunks per 12-vector
    const bool has_ur = it.uref != nullptr;
    auto prefetch = [&](int sg) {
        if (sg >= 0) {
            T *d = s.in[sg % 3];
            const size_t o = (size_t)b * (N + 2) * NX + (size_t)sg * NX;
            const size_t ou = ((size_t)b * (N + 1) + (sg <= N ? sg : 0)) * NX;
            const int nrow = sg <= N ? (has_ur ? 6 : 5) : 3;
            for (int c = lane; c < nrow * RCH; c += WS) {
                const int q = c / RCH, e = (c - q * RCH) * EPC;
                const T *src = q == 0 ? it.x + o : q == 1 ? it.lam + o : q == 2 ? it.xref + o
                             : q == 3 ? it.u + ou : q == 4 ? it.feet + ou : it.uref + ou;
                cp_async16(d + 12 * q + e, src + e);
            }
            if (sg <= N && lane == 0) cp_async4(d + FS::IN_CON, it.con + ((size_t)b * (N + 1) + sg) * 4);
        }
        cp_async_commit();
    };
    prefetch(N + 1);
    prefetch(N);
    // LM shift of pdilqr_solve's ladder (the LM instantiation); a plain step compiles it away
    const T rho_b = LM ? (T)it.rho_of(b) : T(0);
    __syncwarp(mask);
    for (int i = N; i >= 0; --i) {
        prefetch(i - 1);
        cp_async_wait<1>();
        __syncwarp(mask);
        const T *cur = s.in[i % 3], *nxt = s.in[(i + 1) % 3];
        const T *x = cur + FS::IN_X, *lam = cur + FS::IN_L, *ln = nxt + FS::IN_L;
        const T *u = cur + FS::IN_U, *feet = cur + FS::IN_F;
        const uint8_t *con = reinterpret_cast<const uint8_t *>(cur + FS::IN_CON);
        const T *ur = has_ur ? cur + FS::IN_UR : nullptr;
        // ---------------- linearise stage i
        SrbdRow<T> row;
        srbd_stage_row<T>(K, x, u, feet, con, ur, r, row, rho_b);
        bad = bad || row.bad || !isfinite(lam[r]);
        T arow[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) arow[j] = (j == r ? T(1) : T(0)) + row.Arow[j];
        if (act) {
            st_row<T, NX, true>(s.A + r * NX, arow);
            st_row<T, NX, true>(s.B + r * NX, row.Brow);
            st_row<T, NX, true>(s.X + r * NX, row.Arow);  // dt Fx (scratch)
            s.c[r] = (x[r] - nxt[FS::IN_X + r]) + dt * row.fr;  // b_i = h(x_i, u_i) - x_{i+1}
        }
        __syncwarp(mask);
        T qr, rr;
        {
            T ATl = T(0), BTl = T(0);
#pragma unroll
            for (int t = 0; t < NX; ++t) { ATl = fma(s.X[t * NX + r], ln[t], ATl); BTl = fma(s.B[t * NX + r], ln[t], BTl); }
            qr = T(K.wx[r]) * (x[r] - cur[FS::IN_XR + r]) + ((ln[r] - lam[r]) + ATl);
            rr = row.rg + BTl;
        }
        // ---------------- element e_i (Eq. 12 with S = 0): A~ = A, P~ = Q, p~ = q,
        //                  C~ = B R^-1 B^T, b~ = b - B R^-1 r.  Folding it into the suffix
        //                  s_{i+1} (A~ = C~ = b~ = 0) by the cheap rule (Eq. 11) needs
        //                  X = M^-1 A~ with M = I + C~ P_{i+1}; by the Woodbury identity
        //                  X = A - B G^-1 B^T P_{i+1} A = A + B K_i = Abar_i (design D7), so the
        //                  combine shares the policy's elimination and C~ is never formed.
        //                  R is block diagonal (one 3x3 SPD block per foot), so R^-1 r is formed
        //                  blockwise in closed form (adjugate) by the three lanes of each foot.
        if (act) {
            st_row<T, NX, true>(s.ZB + r * NX, row.Rrow);
            s.zr[r] = rr;
        }
        __syncwarp(mask);
        {
            const int jf = r / 3, ar = r - 3 * (r / 3), o = 3 * jf;
            const T *Rb = s.ZB + o * NX + o;
            const T a00 = Rb[0], a01 = Rb[1], a02 = Rb[2];
            const T a10 = Rb[NX], a11 = Rb[NX + 1], a12 = Rb[NX + 2];
            const T a20 = Rb[2 * NX], a21 = Rb[2 * NX + 1], a22 = Rb[2 * NX + 2];
            const T c00 = a11 * a22 - a12 * a21, c01 = a02 * a21 - a01 * a22, c02 = a01 * a12 - a02 * a11;
            const T c10 = a12 * a20 - a10 * a22, c11 = a00 * a22 - a02 * a20, c12 = a02 * a10 - a00 * a12;
            const T c20 = a10 * a21 - a11 * a20, c21 = a01 * a20 - a00 * a21, c22 = a00 * a11 - a01 * a10;
            const T det = a00 * c00 + a01 * c10 + a02 * c20;
            // SPD check of the block: leading principal minors a00, a00 a11 - a01 a10, det > 0
            if (!(a00 > T(0)) || !(c22 > T(0)) || !(det > T(0)) || !isfinite(det)) fail = min(fail, i + 1);
            const T q0 = (ar == 0 ? c00 : ar == 1 ? c10 : c20);
            const T q1 = (ar == 0 ? c01 : ar == 1 ? c11 : c21);
            const T q2 = (ar == 0 ? c02 : ar == 1 ? c12 : c22);
            const T zr_r = (q0 * s.zr[o] + q1 * s.zr[o + 1] + q2 * s.zr[o + 2]) / det;
            __syncwarp(mask);
            if (act) s.zr[r] = zr_r;
        }
        __syncwarp(mask);
        const T btr = row_dot<T, NX>(row.Brow, s.zr, T(0));
        if (act) s.bt[r] = s.c[r] - btr;
        // ---------------- policy for stage i from s_{i+1} = (P_{i+1}, p_{i+1})
        T prow[NX];
        ld_row<T, NX, true>(prow, s.P + r * NX);
        {
            T pb[NX];
            zero(pb);
            row_mat<T, NX, NX, NX>(pb, prow, s.B);
            const T g = row_dot<T, NX>(prow, s.c, s.p[r]);
            if (act) { st_row<T, NX, true>(s.V + r * NX, pb); s.g[r] = g; }
        }
        __syncwarp(mask);
        {
            // policy system  G [K | k] = -[H | h]  (G = R + B^T P B SPD, H = B^T P A, h = B^T (p + P b) + r)
            T bcol[NX], pbcol[NX], G[NX], rhs[NX + 2];
            ld_col<T, NX>(bcol, s.B + r, NX);
            ld_col<T, NX>(pbcol, s.V + r, NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) G[j] = row.Rrow[j];
            row_mat<T, NX, NX, NX>(G, bcol, s.V);
            zero(*reinterpret_cast<T(*)[NX]>(rhs));
            row_mat<T, NX, NX, NX>(*reinterpret_cast<T(*)[NX]>(rhs), pbcol, s.A);
            rhs[NX] = row_dot<T, NX>(bcol, s.g, rr);
            rhs[NX + 1] = T(0);
            const T wr = row_dot<T, NX>(prow, s.bt, s.p[r]);   // w = p_{i+1} + P_{i+1} b~_i
            if (act) s.w[r] = wr;
            int pr1;
            const bool ok1 = gauss_jordan<T, WS, NX, NX + 2, false, true>(mask, G, rhs, lane, NX, pr1);
            if (!ok1) fail = min(fail, i + 1);
            if (act) {
                T kr[NX];
#pragma unroll
                for (int j = 0; j < NX; ++j) kr[j] = -rhs[j];
                st_row<T, NX, true>(s.K + r * NX, kr);
                s.k[r] = -rhs[NX];
                if (live) {
                    st_row<T, NX, true>(Kk + (size_t)i * KL::SIZE + KL::K + r * NX, kr);
                    Kk[(size_t)i * KL::SIZE + KL::k + r] = -rhs[NX];
                }
            }
        }
        __syncwarp(mask);
        {
            // closed-loop transition (Abar_i, bbar_i) = (A + B K, B k + b)  (Eq. 14) = X of the combine
            T abar[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) abar[j] = arow[j];
            row_mat<T, NX, NX, NX>(abar, row.Brow, s.K);
            const T bb = row_dot<T, NX>(row.Brow, s.k, s.c[r]);
            if (act) st_row<T, NX, true>(s.X + r * NX, abar);
            if (wr_g) {
                st_row<T, NX, true>(Te + (size_t)i * TP + r * NX, abar);
                Te[(size_t)i * TP + NX * NX + r] = bb;
            }
        }
        __syncwarp(mask);
        {
            T V[NX];
            zero(V);
            row_mat<T, NX, NX, NX>(V, prow, s.X);
            if (act) st_row<T, NX, true>(s.V + r * NX, V);
        }
        T pn;
        {
            T xc[NX];
            ld_col<T, NX>(xc, s.X + r, NX);
            pn = row_dot<T, NX>(xc, s.w, qr);
        }
        __syncwarp(mask);
        T Pn[NX];
        {
            T acol[NX];
            ld_col<T, NX>(acol, s.A + r, NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) Pn[j] = (j == r) ? T(K.wx[r]) : T(0);
            row_mat<T, NX, NX, NX>(Pn, acol, s.V);
        }
        __syncwarp(mask);
        symmetrize_rows<T, NX>(Pn, s.ZB, mask, lane);
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, Pn);
            s.p[r] = pn;
        }
        if (wr_g) {
            st_row<T, NX, true>(Pp + (size_t)i * TP + r * NX, Pn);
            Pp[(size_t)i * TP + NX * NX + r] = pn;
        }
        __syncwarp(mask);
    }
    {
        const T x0 = it.x0[(size_t)b * NX + r];
        bad = bad || !isfinite(x0);
    }
    unsigned vb = bad ? 1u : 0u;
#pragma unroll
    for (int off = WS / 2; off >= 1; off >>= 1) vb |= __shfl_xor_sync(0xffffffffu, vb, off, WS);
    const bool any_bad = vb != 0u;
    if (lane == 0 && live) info_out[b] = any_bad ? -1 : (fail != INT_MAX ? fail : 0);
}

// ------------------------------------------ stage-parallel linearisation record (fused path)
// The linearisation and quadraticisation of stage i depends only on the
// iterate, not on the Riccati recursion, so it runs stage-parallel BEFORE the fold: one thread per
// (instance, stage) evaluates the model once (no per-row divergence, no redundant trig per lane)
// and writes a compact record of the structurally nonzero parts; the fold reads it one stage ahead.
// SRBD structure used (x = [p, Theta, v, w], u = 4 GRFs): dt Fx has nonzero rows 0-2 (dt at column
// 6 + r), 3-5 and 9-11; dt Fu has rows 6-8 (dt/m on the stance feet's diagonal) and 9-11; R is
// block diagonal with one 3x3 block per foot.
struct LinRec {
    static constexpr int FA = 0;     // dt Fx rows 3, 4, 5, 9, 10, 11 (6 x 12)
    static constexpr int FB = 72;    // dt Fu rows 9, 10, 11 (3 x 12)
    static constexpr int C = 108;    // b_i = h(x_i, u_i) - x_{i+1}
    static constexpr int Q = 120;    // q_i = W_x (x - xref) + (lam_{i+1} - lam_i) + dt Fx^T lam_{i+1}
    static constexpr int RV = 132;   // r_i = W_u (u - uref) + barrier gradient + dt Fu^T lam_{i+1}
    static constexpr int BT = 144;   // b~_i = b_i - B R^-1 r_i  (Eq. 12)
    static constexpr int RB = 156;   // R row r: the 3 entries of its foot block (columns 3(r/3)..+2)
    static constexpr int BD = 192;   // dt / m on stance foot j, 0 on a swing foot (B rows 6-8)
    static constexpr int FL = 196;   // flags (int in the first 4 bytes): 1 bad input / pitch guard, 2 R block not SPD
    static constexpr int SIZE = 200;
};

// STAGED = true: records assembled in shared memory and copied out coalesced; false: each thread
// writes its record with 16-byte stores (no shared memory, occupancy set by registers only).
template <typename T, bool STAGED>
__global__ void __launch_bounds__(STAGED ? 64 : 128, STAGED ? 1 : 4) k_srbd_lin_rec(SrbdConst K, SrbdIter<T> it, int B, int N, T *rec) {
    constexpr int NX = 12, RS = LinRec::SIZE, RP = RS + 16 / (int)sizeof(T);
    using LR = LinRec;
    extern __shared__ __align__(16) unsigned char smraw[];
    T *sm = reinterpret_cast<T *>(smraw);
    const long total = (long)B * (N + 1);
    const long base = (long)blockIdx.x * blockDim.x;
    const long g = base + threadIdx.x;
    if (g < total) {
        T *o = STAGED ? sm + (size_t)threadIdx.x * RP : rec + (size_t)g * RS;
        const int b = (int)(g / (N + 1)), i = (int)(g - (long)b * (N + 1));
        const size_t sx = (size_t)b * (N + 2) + i, st = (size_t)g;
        T xv[NX], xn[NX], uv[NX], fe[NX], lv[NX], ln[NX], xr[NX];
        ld_row<T, NX, true>(xv, it.x + sx * NX);
        ld_row<T, NX, true>(xn, it.x + (sx + 1) * NX);
        ld_row<T, NX, true>(lv, it.lam + sx * NX);
        ld_row<T, NX, true>(ln, it.lam + (sx + 1) * NX);
        ld_row<T, NX, true>(xr, it.xref + sx * NX);
        ld_row<T, NX, true>(uv, it.u + st * NX);
        ld_row<T, NX, true>(fe, it.feet + st * NX);
        const uint32_t cw = *reinterpret_cast<const uint32_t *>(it.con + st * 4);
        const uint8_t con[4] = {(uint8_t)(cw & 0xff), (uint8_t)((cw >> 8) & 0xff), (uint8_t)((cw >> 16) & 0xff),
                                (uint8_t)(cw >> 24)};
        T urv[NX];
        if (it.uref) ld_row<T, NX, true>(urv, it.uref + st * NX);
        else zero(urv);
        SrbdEval<T> ev;
        ev.init(K, xv, uv, fe, con);
        T fa[NX];
        ev.f_all(K, xv, fa);
        const T dt = T(K.dt);
        bool bad = !(fabs((double)xv[4]) < kPitchGuard);
#pragma unroll
        for (int k = 0; k < NX; ++k)
            bad = bad || !isfinite(fa[k]) || !isfinite(xv[k]) || !isfinite(uv[k]) || !isfinite(lv[k]);
        // q accumulates dt Fx^T lam_{i+1}, rv accumulates dt Fu^T lam_{i+1}
        T q[NX], rv[NX];
        zero(q);
        zero(rv);
#pragma unroll
        for (int a = 0; a < 3; ++a) q[6 + a] = dt * ln[a];   // rows 0-2: dt at column 6 + r
        const T w0 = xv[9], w1 = xv[10], w2 = xv[11];
        auto put_fa = [&](int k, int row, const T (&v)[NX]) {   // dt * (row of Fx)
            T d[NX];
#pragma unroll
            for (int c = 0; c < NX; ++c) { d[c] = dt * v[c]; q[c] = fma(d[c], ln[row], q[c]); }
            st_row<T, NX, true>(o + LR::FA + k * NX, d);
        };
        {
            T a3[NX], a4[NX], a5[NX];
            zero(a3); zero(a4); zero(a5);
            a3[3] = ev.tp * (ev.cr * w1 - ev.sr * w2);
            a3[4] = (ev.sr * w1 + ev.cr * w2) * (ev.icp * ev.icp);
            a3[9] = T(1); a3[10] = ev.sr * ev.tp; a3[11] = ev.cr * ev.tp;
            a4[3] = -ev.sr * w1 - ev.cr * w2;
            a4[10] = ev.cr; a4[11] = -ev.sr;
            a5[3] = (ev.cr * w1 - ev.sr * w2) * ev.icp;
            a5[4] = (ev.sr * w1 + ev.cr * w2) * ev.sp * (ev.icp * ev.icp);
            a5[10] = ev.sr * ev.icp; a5[11] = ev.cr * ev.icp;
            put_fa(0, 3, a3);
            put_fa(1, 4, a4);
            put_fa(2, 5, a5);
        }
        T bd[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            bd[j] = con[j] ? dt * T(K.imass) : T(0);
#pragma unroll
            for (int a = 0; a < 3; ++a) rv[3 * j + a] = fma(bd[j], ln[6 + a], rv[3 * j + a]);
        }
        st_row<T, 4, true>(o + LR::BD, bd);
        T Bw[3][NX];   // dt Fu rows 9-11 (kept for b~)
        {
            const T *R = ev.R;
            const T t0 = ev.tau[0], t1 = ev.tau[1], t2 = ev.tau[2];
            const T cy = ev.cy, sy = ev.sy, cp = ev.cp, sp = ev.sp, sr = ev.sr, cr = ev.cr;
            const T v0[3] = {T(0), R[2] * t0 + R[5] * t1 + R[8] * t2, -(R[1] * t0 + R[4] * t1 + R[7] * t2)};
            const T dP[9] = {-cy * sp, cy * cp * sr, cy * cp * cr, -sy * sp, sy * cp * sr, sy * cp * cr, -cp, -sp * sr, -sp * cr};
            T v1[3], v2[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                v1[c] = dP[c] * t0 + dP[3 + c] * t1 + dP[6 + c] * t2;
                v2[c] = -R[3 + c] * t0 + R[c] * t1;
            }
            T Iw[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) Iw[c] = T(K.I[3 * c]) * w0 + T(K.I[3 * c + 1]) * w1 + T(K.I[3 * c + 2]) * w2;
            const T Wx[9] = {T(0), -w2, w1, w2, T(0), -w0, -w1, w0, T(0)};
            const T IWx[9] = {T(0), -Iw[2], Iw[1], Iw[2], T(0), -Iw[0], -Iw[1], Iw[0], T(0)};
            const T SF[9] = {T(0), -ev.F[2], ev.F[1], ev.F[2], T(0), -ev.F[0], -ev.F[1], ev.F[0], T(0)};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                T Ii[3], Ma[3], ar[NX], br[NX];
#pragma unroll
                for (int c = 0; c < 3; ++c) Ii[c] = T(K.Iinv[3 * a + c]);
#pragma unroll
                for (int bb = 0; bb < 3; ++bb) Ma[bb] = Ii[0] * R[3 * bb] + Ii[1] * R[3 * bb + 1] + Ii[2] * R[3 * bb + 2];
                zero(ar);
                zero(br);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) ar[cc] = Ma[0] * SF[cc] + Ma[1] * SF[3 + cc] + Ma[2] * SF[6 + cc];
                ar[3] = Ii[0] * v0[0] + Ii[1] * v0[1] + Ii[2] * v0[2];
                ar[4] = Ii[0] * v1[0] + Ii[1] * v1[1] + Ii[2] * v1[2];
                ar[5] = Ii[0] * v2[0] + Ii[1] * v2[1] + Ii[2] * v2[2];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    T s = T(0);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const T WI = Wx[3 * c] * T(K.I[cc]) + Wx[3 * c + 1] * T(K.I[3 + cc]) + Wx[3 * c + 2] * T(K.I[6 + cc]);
                        s += Ii[c] * (WI - IWx[3 * c + cc]);
                    }
                    ar[9 + cc] = -s;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (!con[j]) continue;
                    const T rx = fe[3 * j] - xv[0], ry = fe[3 * j + 1] - xv[1], rz = fe[3 * j + 2] - xv[2];
                    const T Sr[9] = {T(0), -rz, ry, rz, T(0), -rx, -ry, rx, T(0)};
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) br[3 * j + cc] = Ma[0] * Sr[cc] + Ma[1] * Sr[3 + cc] + Ma[2] * Sr[6 + cc];
                }
                put_fa(3 + a, 9 + a, ar);
#pragma unroll
                for (int c = 0; c < NX; ++c) { Bw[a][c] = dt * br[c]; rv[c] = fma(Bw[a][c], ln[9 + a], rv[c]); }
                st_row<T, NX, true>(o + LR::FB + a * NX, Bw[a]);
            }
        }
        // b_i, q_i
        T c[NX];
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            c[k] = (xv[k] - xn[k]) + dt * fa[k];
            q[k] = T(K.wx[k]) * (xv[k] - xr[k]) + ((ln[k] - lv[k]) + q[k]);
        }
        st_row<T, NX, true>(o + LR::C, c);
        st_row<T, NX, true>(o + LR::Q, q);
        // r_i, R blocks and z = R^-1 r per foot block (adjugate; SPD check)
        const T rho = T(it.rho_of(b));
        bool rfail = false;
        T z[NX];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool stance = con[j] != 0;
            const T wu = stance ? T(K.wu_st) : T(K.wu_sw);
            const FootBarrier<T> fb = foot_barrier<T>(K, uv[3 * j], uv[3 * j + 1], uv[3 * j + 2]);
            const T gb[3] = {fb.gx, fb.gy, fb.gz};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                T rg = wu * (uv[3 * j + a] - urv[3 * j + a]);
                if (stance) rg += gb[a];
                rv[3 * j + a] += rg;
            }
            const T hs = stance ? T(1) : T(0);
            const T a00 = wu + rho + hs * fb.hxx, a11 = wu + rho + hs * fb.hyy, a22 = wu + rho + hs * fb.hzz;
            const T a01 = T(0), a02 = hs * fb.hxz, a12 = hs * fb.hyz;
            const T a10 = a01, a20 = a02, a21 = a12;
            const T Rb[3][3] = {{a00, a01, a02}, {a10, a11, a12}, {a20, a21, a22}};
#pragma unroll
            for (int a = 0; a < 3; ++a) st_row<T, 3, false>(o + LR::RB + 3 * (3 * j + a), Rb[a]);
            const T c00 = a11 * a22 - a12 * a21, c01 = a02 * a21 - a01 * a22, c02 = a01 * a12 - a02 * a11;
            const T c10 = a12 * a20 - a10 * a22, c11 = a00 * a22 - a02 * a20, c12 = a02 * a10 - a00 * a12;
            const T c20 = a10 * a21 - a11 * a20, c21 = a01 * a20 - a00 * a21, c22 = a00 * a11 - a01 * a10;
            const T det = a00 * c00 + a01 * c10 + a02 * c20;
            rfail = rfail || !(a00 > T(0)) || !(c22 > T(0)) || !(det > T(0)) || !isfinite(det);
            const T r0 = rv[3 * j], r1 = rv[3 * j + 1], r2 = rv[3 * j + 2];
            z[3 * j] = (c00 * r0 + c01 * r1 + c02 * r2) / det;
            z[3 * j + 1] = (c10 * r0 + c11 * r1 + c12 * r2) / det;
            z[3 * j + 2] = (c20 * r0 + c21 * r1 + c22 * r2) / det;
        }
        st_row<T, NX, true>(o + LR::RV, rv);
        // b~ = b - B R^-1 r  (B rows 0-5 zero, rows 6-8 dt/m on the stance feet, rows 9-11 Bw)
        T bt[NX];
#pragma unroll
        for (int k = 0; k < 6; ++k) bt[k] = c[k];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            T s6 = T(0), s9 = T(0);
#pragma unroll
            for (int j = 0; j < 4; ++j) s6 = fma(bd[j], z[3 * j + a], s6);
#pragma unroll
            for (int t = 0; t < NX; ++t) s9 = fma(Bw[a][t], z[t], s9);
            bt[6 + a] = c[6 + a] - s6;
            bt[9 + a] = c[9 + a] - s9;
        }
        st_row<T, NX, true>(o + LR::BT, bt);
#pragma unroll
        for (int k = LR::FL; k < LR::SIZE; ++k) o[k] = T(0);
        reinterpret_cast<int *>(o + LR::FL)[0] = (bad ? 1 : 0) | (rfail ? 2 : 0);
    }
    if constexpr (!STAGED) return;
    __syncthreads();
    // coalesced copy of the block's records (contiguous in global memory) in 16-byte granules
    const long nrec = total - base < (long)blockDim.x ? total - base : (long)blockDim.x;
    if (nrec <= 0) return;
    constexpr int EPC = 16 / (int)sizeof(T);
    T *dst = rec + (size_t)base * RS;
    for (long e = (long)threadIdx.x * EPC; e < nrec * RS; e += (long)blockDim.x * EPC) {
        const int t = (int)(e / RS), k = (int)(e - (long)t * RS);
        *reinterpret_cast<int4 *>(dst + e) = *reinterpret_cast<const int4 *>(sm + (size_t)t * RP + k);
    }
}

// The same record by two warps per 32 stages (block of 64 threads, no divergence): warp 0 the
// state half (dt Fx rows, q, b, input checks), warp 1 the control half (dt Fu rows, R blocks, r,
// b~ = b - B R^-1 r, SPD check); both evaluate the model's shared terms.  Half the registers of
// k_srbd_lin_rec per thread, twice the resident warps.  Flag words: FL[0] (state), FL[1] (control).
template <typename T>
__global__ void __launch_bounds__(64, sizeof(T) == 4 ? 8 : 4) k_srbd_lin_rec2(SrbdConst K, SrbdIter<T> it, int B, int N, T *rec) {
    constexpr int NX = 12, RS = LinRec::SIZE, RP = RS + 16 / (int)sizeof(T);
    using LR = LinRec;
    extern __shared__ __align__(16) unsigned char smraw[];
    T *sm = reinterpret_cast<T *>(smraw);
    const long total = (long)B * (N + 1);
    const long base = (long)blockIdx.x * 32;
    const int t = threadIdx.x & 31, half = threadIdx.x >> 5;
    const long g = base + t;
    if (g < total) {
        T *o = sm + (size_t)t * RP;
        const int b = (int)(g / (N + 1)), i = (int)(g - (long)b * (N + 1));
        const size_t sx = (size_t)b * (N + 2) + i, st = (size_t)g;
        const T dt = T(K.dt);
        T xv[NX], uv[NX], fe[NX], ln[NX];
        ld_row<T, NX, true>(xv, it.x + sx * NX);
        ld_row<T, NX, true>(uv, it.u + st * NX);
        ld_row<T, NX, true>(fe, it.feet + st * NX);
        ld_row<T, NX, true>(ln, it.lam + (sx + 1) * NX);
        const uint32_t cw = *reinterpret_cast<const uint32_t *>(it.con + st * 4);
        const uint8_t con[4] = {(uint8_t)(cw & 0xff), (uint8_t)((cw >> 8) & 0xff), (uint8_t)((cw >> 16) & 0xff),
                                (uint8_t)(cw >> 24)};
        SrbdEval<T> ev;
        ev.init(K, xv, uv, fe, con);
        T c[NX];
        {
            T xn[NX], fa[NX];
            ld_row<T, NX, true>(xn, it.x + (sx + 1) * NX);
            ev.f_all(K, xv, fa);
#pragma unroll
            for (int k = 0; k < NX; ++k) c[k] = (xv[k] - xn[k]) + dt * fa[k];   // b_i = h(x_i, u_i) - x_{i+1}
            if (half == 0) {
                bool bad = !(fabs((double)xv[4]) < kPitchGuard);
                T lv[NX];
                ld_row<T, NX, true>(lv, it.lam + sx * NX);
#pragma unroll
                for (int k = 0; k < NX; ++k)
                    bad = bad || !isfinite(fa[k]) || !isfinite(xv[k]) || !isfinite(uv[k]) || !isfinite(lv[k]);
                reinterpret_cast<int *>(o + LR::FL)[0] = bad ? 1 : 0;
                st_row<T, NX, true>(o + LR::C, c);
#pragma unroll
                for (int k = 0; k < NX; ++k) c[k] = ln[k] - lv[k];   // state half: c now holds lam_{i+1} - lam_i
            }
        }
        const T w0 = xv[9], w1 = xv[10], w2 = xv[11];
        if (half == 0) {
            // ---- state half: dt Fx rows 3-5, 9-11 and q = W_x (x - xref) + (lam_{i+1} - lam_i) + dt Fx^T lam_{i+1}
            T q[NX];
            zero(q);
#pragma unroll
            for (int a = 0; a < 3; ++a) q[6 + a] = dt * ln[a];
            auto put_fa = [&](int k, int row, const T (&v)[NX]) {
                T d[NX];
#pragma unroll
                for (int cc = 0; cc < NX; ++cc) { d[cc] = dt * v[cc]; q[cc] = fma(d[cc], ln[row], q[cc]); }
                st_row<T, NX, true>(o + LR::FA + k * NX, d);
            };
            {
                T a3[NX], a4[NX], a5[NX];
                zero(a3); zero(a4); zero(a5);
                a3[3] = ev.tp * (ev.cr * w1 - ev.sr * w2);
                a3[4] = (ev.sr * w1 + ev.cr * w2) * (ev.icp * ev.icp);
                a3[9] = T(1); a3[10] = ev.sr * ev.tp; a3[11] = ev.cr * ev.tp;
                a4[3] = -ev.sr * w1 - ev.cr * w2;
                a4[10] = ev.cr; a4[11] = -ev.sr;
                a5[3] = (ev.cr * w1 - ev.sr * w2) * ev.icp;
                a5[4] = (ev.sr * w1 + ev.cr * w2) * ev.sp * (ev.icp * ev.icp);
                a5[10] = ev.sr * ev.icp; a5[11] = ev.cr * ev.icp;
                put_fa(0, 3, a3);
                put_fa(1, 4, a4);
                put_fa(2, 5, a5);
            }
            {
                const T *R = ev.R;
                const T t0 = ev.tau[0], t1 = ev.tau[1], t2 = ev.tau[2];
                const T cy = ev.cy, sy = ev.sy, cp = ev.cp, sp = ev.sp, sr = ev.sr, cr = ev.cr;
                const T v0[3] = {T(0), R[2] * t0 + R[5] * t1 + R[8] * t2, -(R[1] * t0 + R[4] * t1 + R[7] * t2)};
                const T dP[9] = {-cy * sp, cy * cp * sr, cy * cp * cr, -sy * sp, sy * cp * sr, sy * cp * cr, -cp, -sp * sr, -sp * cr};
                T v1[3], v2[3];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    v1[cc] = dP[cc] * t0 + dP[3 + cc] * t1 + dP[6 + cc] * t2;
                    v2[cc] = -R[3 + cc] * t0 + R[cc] * t1;
                }
                T Iw[3];
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) Iw[cc] = T(K.I[3 * cc]) * w0 + T(K.I[3 * cc + 1]) * w1 + T(K.I[3 * cc + 2]) * w2;
                const T Wx[9] = {T(0), -w2, w1, w2, T(0), -w0, -w1, w0, T(0)};
                const T IWx[9] = {T(0), -Iw[2], Iw[1], Iw[2], T(0), -Iw[0], -Iw[1], Iw[0], T(0)};
                const T SF[9] = {T(0), -ev.F[2], ev.F[1], ev.F[2], T(0), -ev.F[0], -ev.F[1], ev.F[0], T(0)};
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    T Ii[3], Ma[3], ar[NX];
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) Ii[cc] = T(K.Iinv[3 * a + cc]);
#pragma unroll
                    for (int bb = 0; bb < 3; ++bb) Ma[bb] = Ii[0] * R[3 * bb] + Ii[1] * R[3 * bb + 1] + Ii[2] * R[3 * bb + 2];
                    zero(ar);
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) ar[cc] = Ma[0] * SF[cc] + Ma[1] * SF[3 + cc] + Ma[2] * SF[6 + cc];
                    ar[3] = Ii[0] * v0[0] + Ii[1] * v0[1] + Ii[2] * v0[2];
                    ar[4] = Ii[0] * v1[0] + Ii[1] * v1[1] + Ii[2] * v1[2];
                    ar[5] = Ii[0] * v2[0] + Ii[1] * v2[1] + Ii[2] * v2[2];
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) {
                        T sacc = T(0);
#pragma unroll
                        for (int e = 0; e < 3; ++e) {
                            const T WI = Wx[3 * e] * T(K.I[cc]) + Wx[3 * e + 1] * T(K.I[3 + cc]) + Wx[3 * e + 2] * T(K.I[6 + cc]);
                            sacc += Ii[e] * (WI - IWx[3 * e + cc]);
                        }
                        ar[9 + cc] = -sacc;
                    }
                    put_fa(3 + a, 9 + a, ar);
                }
            }
            T xr[NX];
            ld_row<T, NX, true>(xr, it.xref + sx * NX);
#pragma unroll
            for (int k = 0; k < NX; ++k) q[k] = T(K.wx[k]) * (xv[k] - xr[k]) + (c[k] + q[k]);   // c holds lam_{i+1} - lam_i
            st_row<T, NX, true>(o + LR::Q, q);
        } else {
            // ---- control half: dt Fu rows 9-11, R blocks, r, b~
            T rv[NX], bd[4];
            zero(rv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                bd[j] = con[j] ? dt * T(K.imass) : T(0);
#pragma unroll
                for (int a = 0; a < 3; ++a) rv[3 * j + a] = fma(bd[j], ln[6 + a], rv[3 * j + a]);
            }
            st_row<T, 4, true>(o + LR::BD, bd);
            T Bw[3][NX];
            {
                const T *R = ev.R;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    T Ii[3], Ma[3], br[NX];
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) Ii[cc] = T(K.Iinv[3 * a + cc]);
#pragma unroll
                    for (int bb = 0; bb < 3; ++bb) Ma[bb] = Ii[0] * R[3 * bb] + Ii[1] * R[3 * bb + 1] + Ii[2] * R[3 * bb + 2];
                    zero(br);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (!con[j]) continue;
                        const T rx = fe[3 * j] - xv[0], ry = fe[3 * j + 1] - xv[1], rz = fe[3 * j + 2] - xv[2];
                        const T Sr[9] = {T(0), -rz, ry, rz, T(0), -rx, -ry, rx, T(0)};
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) br[3 * j + cc] = Ma[0] * Sr[cc] + Ma[1] * Sr[3 + cc] + Ma[2] * Sr[6 + cc];
                    }
#pragma unroll
                    for (int cc = 0; cc < NX; ++cc) { Bw[a][cc] = dt * br[cc]; rv[cc] = fma(Bw[a][cc], ln[9 + a], rv[cc]); }
                    st_row<T, NX, true>(o + LR::FB + a * NX, Bw[a]);
                }
            }
            T urv[NX];
            if (it.uref) ld_row<T, NX, true>(urv, it.uref + st * NX);
            else zero(urv);
            const T rho = T(it.rho_of(b));
            bool rfail = false;
            T z[NX];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool stance = con[j] != 0;
                const T wu = stance ? T(K.wu_st) : T(K.wu_sw);
                const FootBarrier<T> fb = foot_barrier<T>(K, uv[3 * j], uv[3 * j + 1], uv[3 * j + 2]);
                const T gb[3] = {fb.gx, fb.gy, fb.gz};
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    T rg = wu * (uv[3 * j + a] - urv[3 * j + a]);
                    if (stance) rg += gb[a];
                    rv[3 * j + a] += rg;
                }
                const T hs = stance ? T(1) : T(0);
                const T a00 = wu + rho + hs * fb.hxx, a11 = wu + rho + hs * fb.hyy, a22 = wu + rho + hs * fb.hzz;
                const T a01 = T(0), a02 = hs * fb.hxz, a12 = hs * fb.hyz;
                const T a10 = a01, a20 = a02, a21 = a12;
                const T Rb[3][3] = {{a00, a01, a02}, {a10, a11, a12}, {a20, a21, a22}};
#pragma unroll
                for (int a = 0; a < 3; ++a) st_row<T, 3, false>(o + LR::RB + 3 * (3 * j + a), Rb[a]);
                const T c00 = a11 * a22 - a12 * a21, c01 = a02 * a21 - a01 * a22, c02 = a01 * a12 - a02 * a11;
                const T c10 = a12 * a20 - a10 * a22, c11 = a00 * a22 - a02 * a20, c12 = a02 * a10 - a00 * a12;
                const T c20 = a10 * a21 - a11 * a20, c21 = a01 * a20 - a00 * a21, c22 = a00 * a11 - a01 * a10;
                const T det = a00 * c00 + a01 * c10 + a02 * c20;
                rfail = rfail || !(a00 > T(0)) || !(c22 > T(0)) || !(det > T(0)) || !isfinite(det);
                const T r0 = rv[3 * j], r1 = rv[3 * j + 1], r2 = rv[3 * j + 2];
                z[3 * j] = (c00 * r0 + c01 * r1 + c02 * r2) / det;
                z[3 * j + 1] = (c10 * r0 + c11 * r1 + c12 * r2) / det;
                z[3 * j + 2] = (c20 * r0 + c21 * r1 + c22 * r2) / det;
            }
            st_row<T, NX, true>(o + LR::RV, rv);
            T bt[NX];
#pragma unroll
            for (int k = 0; k < 6; ++k) bt[k] = c[k];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                T s6 = T(0), s9 = T(0);
#pragma unroll
                for (int j = 0; j < 4; ++j) s6 = fma(bd[j], z[3 * j + a], s6);
#pragma unroll
                for (int tt = 0; tt < NX; ++tt) s9 = fma(Bw[a][tt], z[tt], s9);
                bt[6 + a] = c[6 + a] - s6;
                bt[9 + a] = c[9 + a] - s9;
            }
            st_row<T, NX, true>(o + LR::BT, bt);
            reinterpret_cast<int *>(o + LR::FL)[1] = rfail ? 2 : 0;
            if constexpr (sizeof(T) == 4) { o[LR::FL + 2] = T(0); o[LR::FL + 3] = T(0); }
            else { o[LR::FL + 1] = T(0); o[LR::FL + 2] = T(0); o[LR::FL + 3] = T(0); }
        }
    }
    __syncthreads();
    const long nrec = total - base < 32 ? total - base : 32;
    if (nrec <= 0) return;
    constexpr int EPC = 16 / (int)sizeof(T);
    T *dst = rec + (size_t)base * RS;
    for (long e = (long)threadIdx.x * EPC; e < nrec * RS; e += (long)blockDim.x * EPC) {
        const int tt = (int)(e / RS), k = (int)(e - (long)tt * RS);
        *reinterpret_cast<int4 *>(dst + e) = *reinterpret_cast<const int4 *>(sm + (size_t)tt * RP + k);
    }
}

// Per-worker shared memory of the record-fed fold: matrices of the recursion plus a two-slot ring
// of linearisation records (stage i-1 lands while stage i is processed).
template <typename T>
struct FoldRecSmem {
    T in[2][LinRec::SIZE];
    T P[144], A[144], B[144], X[144], V[144], K[144];
    T p[12], g[12], w[12], k[12];
};

// k_srbd_bwd_fold fed by k_srbd_lin_rec: the same recursion (policy, D7 combine, Eq. 5 rows,
// Eq. 11-14) without the linearisation in the sequential loop.
template <typename T, int MINB, int TPB = 64>
__global__ void __launch_bounds__(TPB, MINB * 128 / TPB) k_srbd_bwd_fold_rec(SrbdConst K, SrbdIter<T> it, int B, int N,
                                                                             LqWork<T> ws, const T *rec, int32_t *info_out) {
    constexpr int WS = 16, NX = 12;
    constexpr int TP = TE<NX>::SIZE;
    using KL = KE<NX, NX>;
    using LR = LinRec;
    extern __shared__ __align__(16) unsigned char smraw[];
    FoldRecSmem<T> &s = reinterpret_cast<FoldRecSmem<T> *>(smraw)[threadIdx.x / WS];
    const int lane = worker_lane<WS>();
    const unsigned mask = 0xffffffffu;
    const int b_raw = blockIdx.x * (blockDim.x / WS) + threadIdx.x / WS;
    if (__all_sync(0xffffffffu, b_raw >= B)) return;
    const bool live = b_raw < B;
    const int b = live ? b_raw : B - 1;
    const int r = lane < NX ? lane : 0;
    const bool act = lane < NX;
    const bool wr_g = act && live;
    const T *xb = it.x + (size_t)b * (N + 2) * NX;
    const T *lb = it.lam + (size_t)b * (N + 2) * NX;
    const T *xrb = it.xref + (size_t)b * (N + 2) * NX;
    const T *rb = rec + (size_t)b * (N + 1) * LR::SIZE;
    T *Pp = ws.Pp + (size_t)b * (N + 2) * TP;
    T *Kk = ws.Kk + (size_t)b * (N + 1) * KL::SIZE;
    T *Te = ws.tel + (size_t)b * (N + 1) * TP;
    const T dt = T(K.dt);
    bool bad = false;
    int fail = INT_MAX;
    constexpr int EPC = 16 / (int)sizeof(T), NCH = LR::SIZE / EPC;
    auto prefetch = [&](int sg) {
        if (sg >= 0) {
            T *d = s.in[sg & 1];
            const T *src = rb + (size_t)sg * LR::SIZE;
            for (int c = lane; c < NCH; c += WS) cp_async16(d + c * EPC, src + c * EPC);
        }
        cp_async_commit();
    };
    prefetch(N);
    // terminal element e_{N+1} = suffix s_{N+1}: P = W_N, p = W_N (x_{N+1} - xref) - lam_{N+1}  (Eq. 13)
    {
        const T xr = xb[(N + 1) * NX + r], lr = lb[(N + 1) * NX + r];
        T Prow[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) Prow[j] = (j == r) ? T(K.wxt[r]) : T(0);
        const T pr = T(K.wxt[r]) * (xr - xrb[(N + 1) * NX + r]) - lr;
        bad = bad || !isfinite(xr) || !isfinite(lr);
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, Prow);
            s.p[r] = pr;
        }
        if (wr_g) {
            st_row<T, NX, true>(Pp + (size_t)(N + 1) * TP + r * NX, Prow);
            Pp[(size_t)(N + 1) * TP + NX * NX + r] = pr;
        }
    }
    // this lane's rows of the record: dt Fx row (3-5, 9-11), dt Fu row (9-11), R foot block row
    const int fa_row = (r >= 3 && r <= 5) ? r - 3 : (r >= 9 ? r - 6 : 0);
    const bool has_fa = (r >= 3 && r <= 5) || r >= 9;
    const int fb_row = r >= 9 ? r - 9 : 0;
    const bool has_fb = r >= 9;
    const int jf = r / 3, a6 = r - 6;
    for (int i = N; i >= 0; --i) {
        prefetch(i - 1);
        cp_async_wait<1>();
        __syncwarp(mask);
        const T *cur = s.in[i & 1];
        {
            const int fl = reinterpret_cast<const int *>(cur + LR::FL)[0] | reinterpret_cast<const int *>(cur + LR::FL)[1];
            bad = bad || (fl & 1);
            if (fl & 2) fail = min(fail, i + 1);
        }
        T arow[NX], brow[NX], Rrow[NX];
        {
            T fr[NX], fb[NX], bd[4];
            ld_row<T, NX, true>(fr, cur + LR::FA + fa_row * NX);
            ld_row<T, NX, true>(fb, cur + LR::FB + fb_row * NX);
            ld_row<T, 4, true>(bd, cur + LR::BD);
            const T r0 = cur[LR::RB + 3 * r], r1 = cur[LR::RB + 3 * r + 1], r2 = cur[LR::RB + 3 * r + 2];
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                arow[j] = (j == r ? T(1) : T(0)) + (has_fa ? fr[j] : ((j >= 6 && j < 9 && j - 6 == r) ? dt : T(0)));
                brow[j] = has_fb ? fb[j] : ((a6 >= 0 && a6 < 3 && j % 3 == a6) ? bd[j / 3] : T(0));
                const T rj = (j % 3 == 0) ? r0 : (j % 3 == 1) ? r1 : r2;
                Rrow[j] = (j / 3 == jf) ? rj : T(0);
            }
        }
        const T qr = cur[LR::Q + r], rr = cur[LR::RV + r];
        const T *sc = cur + LR::C, *sbt = cur + LR::BT;
        if (act) {
            st_row<T, NX, true>(s.A + r * NX, arow);
            st_row<T, NX, true>(s.B + r * NX, brow);
        }
        __syncwarp(mask);
        // ---------------- policy for stage i from s_{i+1} = (P_{i+1}, p_{i+1}) and the D7 combine
        T prow[NX];
        ld_row<T, NX, true>(prow, s.P + r * NX);
        {
            T pb[NX];
            zero(pb);
            row_mat<T, NX, NX, NX>(pb, prow, s.B);
            const T gv = row_dot<T, NX>(prow, sc, s.p[r]);
            if (act) { st_row<T, NX, true>(s.V + r * NX, pb); s.g[r] = gv; }
        }
        __syncwarp(mask);
        {
            // policy system  G [K | k] = -[H | h]  (G = R + B^T P B SPD, H = B^T P A, h = B^T (p + P b) + r)
            T bcol[NX], pbcol[NX], G[NX], rhs[NX + 2];
            ld_col<T, NX>(bcol, s.B + r, NX);
            ld_col<T, NX>(pbcol, s.V + r, NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) G[j] = Rrow[j];
            row_mat<T, NX, NX, NX>(G, bcol, s.V);
            zero(*reinterpret_cast<T(*)[NX]>(rhs));
            row_mat<T, NX, NX, NX>(*reinterpret_cast<T(*)[NX]>(rhs), pbcol, s.A);
            rhs[NX] = row_dot<T, NX>(bcol, s.g, rr);
            rhs[NX + 1] = T(0);
            const T wr = row_dot<T, NX>(prow, sbt, s.p[r]);   // w = p_{i+1} + P_{i+1} b~_i
            if (act) s.w[r] = wr;
            int pr1;
            const bool ok1 = gauss_jordan<T, WS, NX, NX + 2, false, true>(mask, G, rhs, lane, NX, pr1);
            if (!ok1) fail = min(fail, i + 1);
            if (act) {
                T kr[NX];
#pragma unroll
                for (int j = 0; j < NX; ++j) kr[j] = -rhs[j];
                st_row<T, NX, true>(s.K + r * NX, kr);
                s.k[r] = -rhs[NX];
                if (live) {
                    st_row<T, NX, true>(Kk + (size_t)i * KL::SIZE + KL::K + r * NX, kr);
                    Kk[(size_t)i * KL::SIZE + KL::k + r] = -rhs[NX];
                }
            }
        }
        __syncwarp(mask);
        {
            // closed-loop transition (Abar_i, bbar_i) = (A + B K, B k + b)  (Eq. 14) = X of the combine (D7)
            T abar[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) abar[j] = arow[j];
            row_mat<T, NX, NX, NX>(abar, brow, s.K);
            const T bb = row_dot<T, NX>(brow, s.k, sc[r]);
            if (act) st_row<T, NX, true>(s.X + r * NX, abar);
            if (wr_g) {
                st_row<T, NX, true>(Te + (size_t)i * TP + r * NX, abar);
                Te[(size_t)i * TP + NX * NX + r] = bb;
            }
        }
        __syncwarp(mask);
        {
            T V[NX];
            zero(V);
            row_mat<T, NX, NX, NX>(V, prow, s.X);
            if (act) st_row<T, NX, true>(s.V + r * NX, V);
        }
        T pn;
        {
            T xc[NX];
            ld_col<T, NX>(xc, s.X + r, NX);
            pn = row_dot<T, NX>(xc, s.w, qr);
        }
        __syncwarp(mask);
        T Pn[NX];
        {
            T acol[NX];
            ld_col<T, NX>(acol, s.A + r, NX);
#pragma unroll
            for (int j = 0; j < NX; ++j) Pn[j] = (j == r) ? T(K.wx[r]) : T(0);
            row_mat<T, NX, NX, NX>(Pn, acol, s.V);
        }
        __syncwarp(mask);
        symmetrize_rows<T, NX>(Pn, s.V, mask, lane);
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, Pn);
            s.p[r] = pn;
        }
        if (wr_g) {
            st_row<T, NX, true>(Pp + (size_t)i * TP + r * NX, Pn);
            Pp[(size_t)i * TP + NX * NX + r] = pn;
        }
        __syncwarp(mask);
    }
    {
        const T x0 = it.x0[(size_t)b * NX + r];
        bad = bad || !isfinite(x0);
    }
    unsigned vb = bad ? 1u : 0u;
#pragma unroll
    for (int off = WS / 2; off >= 1; off >>= 1) vb |= __shfl_xor_sync(0xffffffffu, vb, off, WS);
    const bool any_bad = vb != 0u;
    if (lane == 0 && live) info_out[b] = any_bad ? -1 : (fail != INT_MAX ? fail : 0);
}

// ------------------------------------------ record-fed fold, one instance per warp (two lanes per row)
// The recursion of k_srbd_bwd_fold_rec with every 12 x 12 matrix split by COLUMN halves over the
// two half-warps: lane (h, r) = lane 16 h + r owns row r, columns [6h, 6h + 6).  Twice the
// resident warps of the two-instances-per-warp fold for the same batch (the fold is latency-bound:
// one dependent chain per instance), and the products skip the structurally zero rows of B
// (rows 0-5: P B and B^T (P B) over k = 6..11 only).
// Shared-memory matrices have a row stride of 16 (halves at columns 0..5 and 8..13: 16-byte
// aligned half rows).  B and P B are stored with PERMUTED columns (natural column k at position
// (k & 1) * 6 + (k >> 1)), so G = R + B^T P B comes out with the even columns in half 0 and the
// odd ones in half 1: the elimination of column k then only shuffles the columns > k that are
// still live in either half (36 instead of 72 shuffles over the 12 pivots).
template <typename T>
struct FoldWSmem {
    static constexpr int LD = 16, MS = 12 * LD;
    T in[2][LinRec::SIZE];
    T P[MS], A[MS], Bp[MS], PB[MS], X[MS], K[MS];
    T p[12], g[12], w[12], k[12];
};

__device__ __forceinline__ constexpr int fw_st(int j) { return j + (j >= 6 ? 2 : 0); }         // storage column
__device__ __forceinline__ constexpr int fw_perm(int k) { return (k & 1) * 6 + (k >> 1); }     // permuted position

template <typename T>
__device__ __forceinline__ void ld6(T (&d)[6], const T *__restrict__ s) {   // 16-byte aligned source
    if constexpr (sizeof(T) == 4) {
        const float4 a = *reinterpret_cast<const float4 *>(s);
        const float2 c = *reinterpret_cast<const float2 *>(s + 4);
        d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = c.x; d[5] = c.y;
    } else {
#pragma unroll
        for (int j = 0; j < 6; j += 2) {
            const double2 a = *reinterpret_cast<const double2 *>(s + j);
            d[j] = a.x; d[j + 1] = a.y;
        }
    }
}
template <typename T>
__device__ __forceinline__ void st6(T *__restrict__ d, const T (&v)[6]) {   // 16-byte aligned destination
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4 *>(d) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float2 *>(d + 4) = make_float2(v[4], v[5]);
    } else {
#pragma unroll
        for (int j = 0; j < 6; j += 2) *reinterpret_cast<double2 *>(d + j) = make_double2(v[j], v[j + 1]);
    }
}
template <typename T>
__device__ __forceinline__ void ld6u(T (&d)[6], const T *__restrict__ s) {  // 8-byte aligned source (half of a 12-row)
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int j = 0; j < 6; j += 2) {
            const float2 a = *reinterpret_cast<const float2 *>(s + j);
            d[j] = a.x; d[j + 1] = a.y;
        }
    } else {
        ld6<T>(d, s);
    }
}
template <typename T>
__device__ __forceinline__ void st6u(T *__restrict__ d, const T (&v)[6]) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int j = 0; j < 6; j += 2) *reinterpret_cast<float2 *>(d + j) = make_float2(v[j], v[j + 1]);
    } else {
        st6<T>(d, v);
    }
}
// out[j] += sum_{k in [K0, K1)} a[k] Y[k][half j]  (Y rows of stride 16, pointer at the half's first column)
template <typename T, int K0, int K1>
__device__ __forceinline__ void row_mat_h(T (&out)[6], const T (&a)[12], const T *__restrict__ Y) {
#pragma unroll
    for (int k = K0; k < K1; ++k) {
        T y[6];
        ld6<T>(y, Y + k * 16);
#pragma unroll
        for (int j = 0; j < 6; j += 2) ffma2(a[k], a[k], y[j], y[j + 1], out[j], out[j + 1]);
    }
}
// full natural row r of a stride-16 matrix
template <typename T>
__device__ __forceinline__ void ld_row16(T (&d)[12], const T *__restrict__ row) {
    T a[6], c[6];
    ld6<T>(a, row);
    ld6<T>(c, row + 8);
#pragma unroll
    for (int j = 0; j < 6; ++j) { d[j] = a[j]; d[6 + j] = c[j]; }
}

template <typename T, int MINB>
__global__ void __launch_bounds__(64, MINB) k_srbd_bwd_fold_w(SrbdConst K, SrbdIter<T> it, int B, int N, LqWork<T> ws,
                                                              const T *rec, int32_t *info_out) {
    constexpr int NX = 12, LD = 16;
    constexpr int TP = TE<NX>::SIZE;
    using KL = KE<NX, NX>;
    using LR = LinRec;
    extern __shared__ __align__(16) unsigned char smraw[];
    FoldWSmem<T> &s = reinterpret_cast<FoldWSmem<T> *>(smraw)[threadIdx.x / 32];
    const int lane = threadIdx.x & 31, h = lane >> 4, r16 = lane & 15;
    const int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (b >= B) return;   // warp-uniform
    const int r = r16 < NX ? r16 : 0;
    const bool act = r16 < NX;
    const bool act0 = act && h == 0;   // writer of per-row scalars
    const int c0 = 6 * h;              // natural columns [c0, c0 + 6) of this lane
    const int so = 8 * h;              // their storage offset in a stride-16 row
    const int rp = fw_st(fw_perm(r));  // storage column of natural column r in a permuted matrix
    const T *xb = it.x + (size_t)b * (N + 2) * NX;
    const T *lb = it.lam + (size_t)b * (N + 2) * NX;
    const T *xrb = it.xref + (size_t)b * (N + 2) * NX;
    const T *rb = rec + (size_t)b * (N + 1) * LR::SIZE;
    T *Pp = ws.Pp + (size_t)b * (N + 2) * TP;
    T *Kk = ws.Kk + (size_t)b * (N + 1) * KL::SIZE;
    T *Te = ws.tel + (size_t)b * (N + 1) * TP;
    const T dt = T(K.dt);
    bool bad = false;
    int fail = INT_MAX;
    constexpr int EPC = 16 / (int)sizeof(T), NCH = LR::SIZE / EPC;
    auto prefetch = [&](int sg) {
        if (sg >= 0) {
            T *d = s.in[sg & 1];
            const T *src = rb + (size_t)sg * LR::SIZE;
            for (int c = lane; c < NCH; c += 32) cp_async16(d + c * EPC, src + c * EPC);
        }
        cp_async_commit();
    };
    prefetch(N);
    // terminal element e_{N+1}: P = W_N, p = W_N (x_{N+1} - xref) - lam_{N+1}  (Eq. 13)
    {
        const T xr = xb[(N + 1) * NX + r], lr = lb[(N + 1) * NX + r];
        T Ph[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) Ph[j] = (c0 + j == r) ? T(K.wxt[r]) : T(0);
        const T pr = T(K.wxt[r]) * (xr - xrb[(N + 1) * NX + r]) - lr;
        bad = bad || !isfinite(xr) || !isfinite(lr);
        if (act) {
            st6<T>(s.P + r * LD + so, Ph);
            st6u<T>(Pp + (size_t)(N + 1) * TP + r * NX + c0, Ph);
        }
        if (act0) {
            s.p[r] = pr;
            Pp[(size_t)(N + 1) * TP + NX * NX + r] = pr;
        }
    }
    const int fa_row = (r >= 3 && r <= 5) ? r - 3 : (r >= 9 ? r - 6 : 0);
    const bool has_fa = (r >= 3 && r <= 5) || r >= 9;
    const int fb_row = r >= 9 ? r - 9 : 0;
    const bool has_fb = r >= 9;
    const int jf = r / 3, a6 = r - 6;
    for (int i = N; i >= 0; --i) {
        prefetch(i - 1);
        cp_async_wait<1>();
        __syncwarp();
        const T *cur = s.in[i & 1];
        {
            const int fl = reinterpret_cast<const int *>(cur + LR::FL)[0] | reinterpret_cast<const int *>(cur + LR::FL)[1];
            bad = bad || (fl & 1);
            if (fl & 2) fail = min(fail, i + 1);
        }
        // ---------------- this lane's parts of A_i (half row), B_i (full row), R_i (permuted half row)
        T ah[6], brow[NX], Rp[6];
        {
            T fr[6], fb[NX], bd[4];
            ld6u<T>(fr, cur + LR::FA + fa_row * NX + c0);
            ld_row<T, NX, true>(fb, cur + LR::FB + fb_row * NX);
            ld_row<T, 4, true>(bd, cur + LR::BD);
            const T r0 = cur[LR::RB + 3 * r], r1 = cur[LR::RB + 3 * r + 1], r2 = cur[LR::RB + 3 * r + 2];
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                const int jn = c0 + j;
                ah[j] = (jn == r ? T(1) : T(0)) + (has_fa ? fr[j] : ((r < 3 && jn == 6 + r) ? dt : T(0)));
            }
#pragma unroll
            for (int j = 0; j < NX; ++j)
                brow[j] = has_fb ? fb[j] : ((a6 >= 0 && a6 < 3 && j % 3 == a6) ? bd[j / 3] : T(0));
#pragma unroll
            for (int jj = 0; jj < 6; ++jj) {
                const int k = 2 * jj + h;   // natural column of permuted position 6 h + jj
                const int kk = k - 3 * jf;
                Rp[jj] = (kk == 0) ? r0 : (kk == 1) ? r1 : (kk == 2) ? r2 : T(0);
            }
        }
        const T qr = cur[LR::Q + r], rr = cur[LR::RV + r];
        const T *sc = cur + LR::C, *sbt = cur + LR::BT;
        if (act) {
            st6<T>(s.A + r * LD + so, ah);
            T bp[6];
#pragma unroll
            for (int jj = 0; jj < 6; ++jj) bp[jj] = h ? brow[2 * jj + 1] : brow[2 * jj];
            st6<T>(s.Bp + r * LD + so, bp);
        }
        __syncwarp();
        // ---------------- policy for stage i from s_{i+1} = (P_{i+1}, p_{i+1})
        T prow[NX];
        ld_row16<T>(prow, s.P + r * LD);
        {
            T pb[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) pb[j] = T(0);
            row_mat_h<T, 6, 12>(pb, prow, s.Bp + so);          // P B (B rows 0-5 are zero), permuted columns
            const T gv = row_dot<T, NX>(prow, sc, s.p[r]);     // g = p_{i+1} + P_{i+1} b_i
            const T wv = row_dot<T, NX>(prow, sbt, s.p[r]);    // w = p_{i+1} + P_{i+1} b~_i
            if (act) st6<T>(s.PB + r * LD + so, pb);
            if (act0) { s.g[r] = gv; s.w[r] = wv; }
        }
        __syncwarp();
        T x[7];   // right-hand sides: H[r][c0..c0+6), and h[r] in half 0
        T a[6];   // G[r][2 jj + h]
        {
            T bc[6], pbc[NX];
#pragma unroll
            for (int k = 0; k < 6; ++k) bc[k] = s.Bp[(6 + k) * LD + rp];     // B[6 + k][r]
#pragma unroll
            for (int k = 0; k < NX; ++k) pbc[k] = s.PB[k * LD + rp];         // (P B)[k][r]
#pragma unroll
            for (int jj = 0; jj < 6; ++jj) a[jj] = Rp[jj];
#pragma unroll
            for (int k = 0; k < 6; ++k) {                                     // G = R + B^T (P B)
                T y[6];
                ld6<T>(y, s.PB + (6 + k) * LD + so);
#pragma unroll
                for (int j = 0; j < 6; j += 2) ffma2(bc[k], bc[k], y[j], y[j + 1], a[j], a[j + 1]);
            }
            T hh[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) hh[j] = T(0);
            row_mat_h<T, 0, 12>(hh, pbc, s.A + so);                           // H = (P B)^T A
            T hv = rr;                                                          // h = B^T g + r
#pragma unroll
            for (int k = 0; k < 6; ++k) hv = fma(bc[k], s.g[6 + k], hv);
#pragma unroll
            for (int j = 0; j < 6; ++j) x[j] = hh[j];
            x[6] = h == 0 ? hv : T(0);
        }
        {
            // SPD Gauss-Jordan on G [K | k] = -[H | h] (unnormalised sweep, pivot rows scaled at the end)
            bool ok = true;
            T mypiv = T(1);
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                const int hk = k & 1, jk = k >> 1;
                const T own = a[jk];
                const T rk = rcp_rn(own);
                const T ark = __shfl_sync(0xffffffffu, own, 16 * hk + r);
                const T pv = __shfl_sync(0xffffffffu, own, 16 * hk + k);
                const T rpv = __shfl_sync(0xffffffffu, rk, 16 * hk + k);
                ok = ok && (pv > T(0)) && isfinite(pv);
                const bool isp = r16 == k;
                const T f = isp ? T(0) : ark * rpv;
                if (isp) mypiv = pv;
                const int src = 16 * h + k;
#pragma unroll
                for (int jj = 0; jj < 6; ++jj)
                    if (2 * jj + 1 > k) a[jj] = fma(-f, __shfl_sync(0xffffffffu, a[jj], src), a[jj]);
#pragma unroll
                for (int j = 0; j < 6; j += 2) {
                    const T p0 = __shfl_sync(0xffffffffu, x[j], src), p1 = __shfl_sync(0xffffffffu, x[j + 1], src);
                    ffma2(-f, -f, p0, p1, x[j], x[j + 1]);
                }
                x[6] = fma(-f, __shfl_sync(0xffffffffu, x[6], src), x[6]);
            }
            const T inv = rcp_rn(mypiv);
#pragma unroll
            for (int j = 0; j < 7; ++j) x[j] *= -inv;   // [K | k] = -G^-1 [H | h]
            if (!ok) fail = min(fail, i + 1);
        }
        {
            T kh[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) kh[j] = x[j];
            if (act) {
                st6<T>(s.K + r * LD + so, kh);
                st6u<T>(Kk + (size_t)i * KL::SIZE + KL::K + r * NX + c0, kh);
            }
            if (act0) {
                s.k[r] = x[6];
                Kk[(size_t)i * KL::SIZE + KL::k + r] = x[6];
            }
        }
        __syncwarp();
        {
            // closed-loop transition (Abar_i, bbar_i) = (A + B K, B k + b)  (Eq. 14) = X of the D7 combine
            T ab[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) ab[j] = ah[j];
            row_mat_h<T, 0, 12>(ab, brow, s.K + so);
            const T bb = row_dot<T, NX>(brow, s.k, sc[r]);
            if (act) {
                st6<T>(s.X + r * LD + so, ab);
                st6u<T>(Te + (size_t)i * TP + r * NX + c0, ab);
            }
            if (act0) Te[(size_t)i * TP + NX * NX + r] = bb;
        }
        __syncwarp();
        T pn;
        {
            T v[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) v[j] = T(0);
            row_mat_h<T, 0, 12>(v, prow, s.X + so);            // V = P_{i+1} Abar_i
            if (act) st6<T>(s.PB + r * LD + so, v);
            T xc[NX];
#pragma unroll
            for (int k = 0; k < NX; ++k) xc[k] = s.X[k * LD + fw_st(r)];
            pn = row_dot<T, NX>(xc, s.w, qr);                  // p_i = q_i + Abar_i^T w
        }
        __syncwarp();
        T Pn[6];
        {
            T ac[NX];
#pragma unroll
            for (int k = 0; k < NX; ++k) ac[k] = s.A[k * LD + fw_st(r)];
#pragma unroll
            for (int j = 0; j < 6; ++j) Pn[j] = (c0 + j == r) ? T(K.wx[r]) : T(0);
            row_mat_h<T, 0, 12>(Pn, ac, s.PB + so);             // P_i = Q + A^T V
        }
        // re-symmetrise (R22) through the dead Abar buffer
        if (act) st6<T>(s.X + r * LD + so, Pn);
        __syncwarp();
        {
            T ct[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) ct[j] = s.X[(c0 + j) * LD + fw_st(r)];
#pragma unroll
            for (int j = 0; j < 6; ++j) Pn[j] = T(0.5) * (Pn[j] + ct[j]);
        }
        __syncwarp();
        if (act) {
            st6<T>(s.P + r * LD + so, Pn);
            st6u<T>(Pp + (size_t)i * TP + r * NX + c0, Pn);
        }
        if (act0) {
            s.p[r] = pn;
            Pp[(size_t)i * TP + NX * NX + r] = pn;
        }
        __syncwarp();
    }
    {
        const T x0 = it.x0[(size_t)b * NX + r];
        bad = bad || !isfinite(x0);
    }
    const bool any_bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) info_out[b] = any_bad ? -1 : (fail != INT_MAX ? fail : 0);
}

// ------------------------------------- record-fed fold, two rows per lane (five instances per warp)
// The fold is bound by the shared-memory data pipe (LDS / STS / SHFL wavefronts; ncu r3_v1: 88 %
// of peak), not by the FMA pipe: a row-per-lane 12 x 12 product makes every lane load all 144
// entries of the other operand.  Here a worker is 6 lanes, lane l owns rows l and l + 6 of every
// matrix (so every loaded operand row feeds two FFMA2 row updates), a warp carries 5 instances
// (lanes 6 NW .. 31 shadow the last lane and store nothing; NW = 4 or 5), and the products use the SRBD structure of the
// linearisation record: B has zero rows 0-5 (P B and B^T P B over k = 6..11), A = I + dt Fx with
// dt Fx nonzero only in rows 3-5, 9-11 plus dt at (r, 6 + r) for r < 3, so H = (P B)^T A and
// P = Q + A^T V take the identity from registers and only 6 operand rows from shared memory.
// Same recursion as k_srbd_bwd_fold_rec (policy Eq. 5 rows, D7 combine, Eq. 11-14, R22).
// Slice stride (fp32 words) = 8 (mod 32) for 2-4 workers per warp (row loads and the 6-lane column
// loads of the workers hit disjoint banks), 4 (mod 32) for 5 workers (row loads disjoint).
template <typename T, int NW>
struct FoldR2Smem {
    T in[2][LinRec::SIZE];
    T P[144], B6[72], PB[144], K[144], X[144];
    T p[12], w[12], k[12];
    T pad[NW <= 4 ? 12 : 8];
};

// CP (stance compaction): the controls of a swing foot have zero columns in B, so they decouple
// from the policy system (G block diagonal: the stance block and the swing feet's R blocks, H = 0 and
// K = 0 on the swing rows, k = -R^-1 r there).  Per stage and instance the feet are permuted stance
// first (B's columns permuted when stored, so P B, G, H, h come out permuted), the elimination runs
// over the first 3 ns pivots only (ns = stance feet; the warp's maximum), and K, k are written back in
// the natural control order.  Same arithmetic on every element that is not structurally zero.
template <typename T, int NW, bool CP = true>
__global__ void __launch_bounds__(32, 6) k_srbd_bwd_fold_r2(SrbdConst K, SrbdIter<T> it, int B, int N, LqWork<T> ws,
                                                           const T *rec, int32_t *info_out) {
    constexpr int NX = 12, NL = 6 * NW;
    constexpr int TP = TE<NX>::SIZE;
    using KL = KE<NX, NX>;
    using LR = LinRec;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int L = threadIdx.x & 31;
    const int w = L < NL ? L / 6 : NW - 1;
    const int l = L < NL ? L - 6 * w : 5;
    const bool lane_act = L < NL;
    FoldR2Smem<T, NW> &s = reinterpret_cast<FoldR2Smem<T, NW> *>(smraw)[(threadIdx.x >> 5) * NW + w];
    const int b_raw = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NW + w;
    if (__all_sync(0xffffffffu, b_raw >= B)) return;
    const bool live = b_raw < B;
    const int b = live ? b_raw : B - 1;
    const bool act = lane_act && live;        // smem + global writer
    const int r0 = l, r1 = l + 6;             // this lane's rows
    const int wb = 6 * w;                     // first lane of the worker
    const T *xb = it.x + (size_t)b * (N + 2) * NX;
    const T *lb = it.lam + (size_t)b * (N + 2) * NX;
    const T *xrb = it.xref + (size_t)b * (N + 2) * NX;
    const T *rb = rec + (size_t)b * (N + 1) * LR::SIZE;
    T *Pp = ws.Pp + (size_t)b * (N + 2) * TP;
    T *Kk = ws.Kk + (size_t)b * (N + 1) * KL::SIZE;
    T *Te = ws.tel + (size_t)b * (N + 1) * TP;
    const T dt = T(K.dt);
    bool bad = false;
    int fail = INT_MAX;
    constexpr int EPC = 16 / (int)sizeof(T), NCH = LR::SIZE / EPC;
    auto prefetch = [&](int sg) {
        if (sg >= 0 && lane_act) {
            T *d = s.in[sg & 1];
            const T *src = rb + (size_t)sg * LR::SIZE;
            for (int c = l; c < NCH; c += 6) cp_async16(d + c * EPC, src + c * EPC);
        }
        cp_async_commit();
    };
    prefetch(N);
    // terminal element e_{N+1}: P = W_N, p = W_N (x_{N+1} - xref) - lam_{N+1}  (Eq. 13)
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
        const int r = l + 6 * sl;
        const T xr = xb[(N + 1) * NX + r], lr = lb[(N + 1) * NX + r];
        T Prow[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) Prow[j] = (j == r) ? T(K.wxt[r]) : T(0);
        const T pr = T(K.wxt[r]) * (xr - xrb[(N + 1) * NX + r]) - lr;
        bad = bad || !isfinite(xr) || !isfinite(lr);
        if (act) {
            st_row<T, NX, true>(s.P + r * NX, Prow);
            s.p[r] = pr;
            st_row<T, NX, true>(Pp + (size_t)(N + 1) * TP + r * NX, Prow);
            Pp[(size_t)(N + 1) * TP + NX * NX + r] = pr;
        }
    }
    const bool lhi = l >= 3;                  // rows l (3..5) and l + 6 (9..11) have dt Fx rows
    const int fa0 = lhi ? l - 3 : 0, fa1 = lhi ? l : 0;
    for (int i = N; i >= 0; --i) {
        prefetch(i - 1);
        cp_async_wait<1>();
        __syncwarp();
        const T *cur = s.in[i & 1];
        {
            const int fl = reinterpret_cast<const int *>(cur + LR::FL)[0] | reinterpret_cast<const int *>(cur + LR::FL)[1];
            bad = bad || (fl & 1);
            if (fl & 2) fail = min(fail, i + 1);
        }
        // B row l + 6 (rows 6-8: dt/m on the stance feet' diagonal, 9-11 the record's dt Fu rows)
        T b1[NX], bd[4];
        int perm = 0xE4, ncm = NX;   // foot of permuted position q = (perm >> 2q) & 3 (identity without CP)
        {
            T fb[NX];
            ld_row<T, NX, true>(fb, cur + LR::FB + (lhi ? l - 3 : 0) * NX);
            ld_row<T, 4, true>(bd, cur + LR::BD);
#pragma unroll
            for (int j = 0; j < NX; ++j) b1[j] = lhi ? fb[j] : ((j % 3 == l) ? bd[j / 3] : T(0));
            if constexpr (CP) {
                int ns = 0, q = 0;
                perm = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (bd[j] != T(0)) { perm |= j << (2 * q); ++q; ++ns; }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (bd[j] == T(0)) { perm |= j << (2 * q); ++q; }
                ncm = __reduce_max_sync(0xffffffffu, 3 * ns);
                T bp[NX];
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const int fq = (perm >> (2 * qq)) & 3;
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        bp[3 * qq + a] = fq == 0 ? b1[a] : fq == 1 ? b1[3 + a] : fq == 2 ? b1[6 + a] : b1[9 + a];
                }
                if (act) st_row<T, NX, true>(s.B6 + l * NX, bp);
            } else {
                if (act) st_row<T, NX, true>(s.B6 + l * NX, b1);
            }
        }
        // this lane's compacted rows c0 = l, c1 = l + 6 are the controls o0, o1 (identity without CP)
        const int o0 = 3 * ((perm >> (2 * (l / 3))) & 3) + l % 3;
        const int o1 = 3 * ((perm >> (2 * (2 + l / 3))) & 3) + l % 3;
        __syncwarp();
        // ---------------- P B (rows 0-5 of B are zero) and w = p + P b~
        {
            T pr0[NX], pr1[NX], pb0[NX], pb1[NX];
            ld_row<T, NX, true>(pr0, s.P + r0 * NX);
            ld_row<T, NX, true>(pr1, s.P + r1 * NX);
            zero(pb0);
            zero(pb1);
#pragma unroll
            for (int k = 6; k < 12; ++k) {
                T y[NX];
                ld_row<T, NX, true>(y, s.B6 + (k - 6) * NX);
#pragma unroll
                for (int j = 0; j < NX; ++j) ffma2(pr0[k], pr1[k], y[j], y[j], pb0[j], pb1[j]);
            }
            T bt[NX];
            ld_row<T, NX, true>(bt, cur + LR::BT);
            T w0 = s.p[r0], w1 = s.p[r1];
#pragma unroll
            for (int k = 0; k < NX; ++k) ffma2(pr0[k], pr1[k], bt[k], bt[k], w0, w1);
            if (act) {
                st_row<T, NX, true>(s.PB + r0 * NX, pb0);
                st_row<T, NX, true>(s.PB + r1 * NX, pb1);
                s.w[r0] = w0;
                s.w[r1] = w1;
            }
        }
        __syncwarp();
        // ---------------- policy system  G [K | k] = -[H | h]:  G = R + (P B)^T B, H = (P B)^T A,
        //                  h = r + B^T p + (P B)^T b  (P symmetric)
        T a0[NX], a1[NX], x0[NX + 1], x1[NX + 1];
        {
            T pc0[NX], pc1[NX];
#pragma unroll
            for (int k = 0; k < NX; ++k) { pc0[k] = s.PB[k * NX + r0]; pc1[k] = s.PB[k * NX + r1]; }
            {   // R rows (block diagonal, 3 x 3 per foot; the permutation keeps foot blocks together)
                const int j0 = r0 / 3, j1 = r1 / 3;
#pragma unroll
                for (int j = 0; j < NX; ++j) {
                    a0[j] = (j / 3 == j0) ? cur[LR::RB + 3 * o0 + (j % 3)] : T(0);
                    a1[j] = (j / 3 == j1) ? cur[LR::RB + 3 * o1 + (j % 3)] : T(0);
                }
            }
#pragma unroll
            for (int k = 6; k < 12; ++k) {
                T y[NX];
                ld_row<T, NX, true>(y, s.B6 + (k - 6) * NX);
#pragma unroll
                for (int j = 0; j < NX; ++j) ffma2(pc0[k], pc1[k], y[j], y[j], a0[j], a1[j]);
            }
            // H: identity part and the dt at (k, 6 + k), k < 3, from registers; dt Fx rows 3-5, 9-11 from the record
#pragma unroll
            for (int j = 0; j < NX; ++j) { x0[j] = pc0[j]; x1[j] = pc1[j]; }
#pragma unroll
            for (int k = 0; k < 3; ++k) ffma2(dt, dt, pc0[k], pc1[k], x0[6 + k], x1[6 + k]);
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                const int k = t < 3 ? 3 + t : 6 + t;
                T y[NX];
                ld_row<T, NX, true>(y, cur + LR::FA + t * NX);
#pragma unroll
                for (int j = 0; j < NX; ++j) ffma2(pc0[k], pc1[k], y[j], y[j], x0[j], x1[j]);
            }
            // h = r + (P B)^T b + B^T p: B^T p over rows 6-8 (one stance term per row) and 9-11 (record)
            T cv[NX], pv[NX];
            ld_row<T, NX, true>(cv, cur + LR::C);
            ld_row<T, NX, true>(pv, s.p);
            T h0 = cur[LR::RV + o0], h1 = cur[LR::RV + o1];
#pragma unroll
            for (int k = 0; k < NX; ++k) ffma2(pc0[k], pc1[k], cv[k], cv[k], h0, h1);
            {
                const T bdj0 = cur[LR::BD + o0 / 3], bdj1 = cur[LR::BD + o1 / 3];
                h0 = fma(bdj0, (o0 % 3 == 0) ? pv[6] : (o0 % 3 == 1) ? pv[7] : pv[8], h0);
                h1 = fma(bdj1, (o1 % 3 == 0) ? pv[6] : (o1 % 3 == 1) ? pv[7] : pv[8], h1);
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const T fb0 = cur[LR::FB + a * NX + o0], fb1 = cur[LR::FB + a * NX + o1];
                    ffma2(fb0, fb1, pv[9 + a], pv[9 + a], h0, h1);
                }
            }
            x0[NX] = h0;
            x1[NX] = h1;
        }
        {
            // SPD Gauss-Jordan, unnormalised sweep; pivot k lives in lane k % 6, slot k / 6.  The pivot
            // count NP is a compile-time bound per branch (6: every instance of the warp has at most two
            // stance feet; 12 otherwise), so neither loop carries a branch.
            bool ok = true;
            // rows that never pivot (swing rows beyond the warp's last pivot) keep their diagonal
            T piv0 = CP ? a0[0] : T(1), piv1 = CP ? a1[0] : T(1);
            if constexpr (CP) {
#pragma unroll
                for (int j = 1; j < NX; ++j) { piv0 = (j == r0) ? a0[j] : piv0; piv1 = (j == r1) ? a1[j] : piv1; }
            }
            auto gj = [&](auto np_tag) {
                constexpr int NP = decltype(np_tag)::value;
#pragma unroll
                for (int k = 0; k < NP; ++k) {
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
                    for (int j = k + 1; j < NP; ++j) {   // columns >= NP are zero in the rows that pivot
                        const T pj = __shfl_sync(0xffffffffu, ps == 0 ? a0[j] : a1[j], src);
                        ffma2(-f0, -f1, pj, pj, a0[j], a1[j]);
                    }
#pragma unroll
                    for (int j = 0; j <= NX; ++j) {
                        const T pj = __shfl_sync(0xffffffffu, ps == 0 ? x0[j] : x1[j], src);
                        ffma2(-f0, -f1, pj, pj, x0[j], x1[j]);
                    }
                }
            };
            if (CP && ncm <= 6) gj(std::integral_constant<int, 6>{});
            else gj(std::integral_constant<int, NX>{});
            const T i0 = -rcp_rn(piv0), i1 = -rcp_rn(piv1);
#pragma unroll
            for (int j = 0; j <= NX; ++j) { x0[j] *= i0; x1[j] *= i1; }   // [K | k] = -G^-1 [H | h]
            if (!ok) fail = min(fail, i + 1);
        }
        if (act) {
            T kr0[NX], kr1[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) { kr0[j] = x0[j]; kr1[j] = x1[j]; }
            st_row<T, NX, true>(s.K + o0 * NX, kr0);
            st_row<T, NX, true>(s.K + o1 * NX, kr1);
            s.k[o0] = x0[NX];
            s.k[o1] = x1[NX];
            st_row<T, NX, true>(Kk + (size_t)i * KL::SIZE + KL::K + o0 * NX, kr0);
            st_row<T, NX, true>(Kk + (size_t)i * KL::SIZE + KL::K + o1 * NX, kr1);
            Kk[(size_t)i * KL::SIZE + KL::k + o0] = x0[NX];
            Kk[(size_t)i * KL::SIZE + KL::k + o1] = x1[NX];
        }
        __syncwarp();
        {
            // closed-loop transition (Abar_i, bbar_i) = (A + B K, B k + b)  (Eq. 14) = X of the D7 combine;
            // rows 0-5 of B are zero: Abar row l = A row l
            T ab0[NX], ab1[NX];
            {
                T f0[NX], f1[NX];
                ld_row<T, NX, true>(f0, cur + LR::FA + fa0 * NX);
                ld_row<T, NX, true>(f1, cur + LR::FA + fa1 * NX);
#pragma unroll
                for (int j = 0; j < NX; ++j) {
                    ab0[j] = (j == r0 ? T(1) : T(0)) + (lhi ? f0[j] : ((j == 6 + l) ? dt : T(0)));
                    ab1[j] = (j == r1 ? T(1) : T(0)) + (lhi ? f1[j] : T(0));
                }
            }
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                T y[NX];
                ld_row<T, NX, true>(y, s.K + k * NX);
#pragma unroll
                for (int j = 0; j < NX; j += 2) ffma2(b1[k], b1[k], y[j], y[j + 1], ab1[j], ab1[j + 1]);
            }
            const T cb0 = cur[LR::C + r0];
            const T bb1 = row_dot<T, NX>(b1, s.k, cur[LR::C + r1]);
            if (act) {
                st_row<T, NX, true>(s.X + r0 * NX, ab0);
                st_row<T, NX, true>(s.X + r1 * NX, ab1);
                st_row<T, NX, true>(Te + (size_t)i * TP + r0 * NX, ab0);
                st_row<T, NX, true>(Te + (size_t)i * TP + r1 * NX, ab1);
                Te[(size_t)i * TP + NX * NX + r0] = cb0;
                Te[(size_t)i * TP + NX * NX + r1] = bb1;
            }
        }
        __syncwarp();
        T pn0, pn1;
        {
            // V = P_{i+1} Abar_i (into the dead P B buffer), p_i = q_i + Abar_i^T w
            T pr0[NX], pr1[NX], v0[NX], v1[NX];
            ld_row<T, NX, true>(pr0, s.P + r0 * NX);
            ld_row<T, NX, true>(pr1, s.P + r1 * NX);
            zero(v0);
            zero(v1);
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                T y[NX];
                ld_row<T, NX, true>(y, s.X + k * NX);
#pragma unroll
                for (int j = 0; j < NX; ++j) ffma2(pr0[k], pr1[k], y[j], y[j], v0[j], v1[j]);
            }
            if (act) {
                st_row<T, NX, true>(s.PB + r0 * NX, v0);
                st_row<T, NX, true>(s.PB + r1 * NX, v1);
            }
            T wv[NX];
            ld_row<T, NX, true>(wv, s.w);
            pn0 = cur[LR::Q + r0];
            pn1 = cur[LR::Q + r1];
#pragma unroll
            for (int k = 0; k < NX; ++k) ffma2(s.X[k * NX + r0], s.X[k * NX + r1], wv[k], wv[k], pn0, pn1);
        }
        __syncwarp();
        T P0[NX], P1[NX];
        {
            // P_i = Q + A^T V = Q + V + dt V[r - 6] (rows 6-8) + sum over the dt Fx rows t of dt Fx[t][r] V[t]
            ld_row<T, NX, true>(P0, s.PB + r0 * NX);
            ld_row<T, NX, true>(P1, s.PB + r1 * NX);
            {
                const T e1 = l < 3 ? dt : T(0);
#pragma unroll
                for (int j = 0; j < NX; ++j) P1[j] = fma(e1, P0[j], P1[j]);   // uses V row l (= r0) before Q is added
            }
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                const int k = t < 3 ? 3 + t : 6 + t;
                const T c0v = cur[LR::FA + t * NX + r0], c1v = cur[LR::FA + t * NX + r1];
                T y[NX];
                ld_row<T, NX, true>(y, s.PB + k * NX);
#pragma unroll
                for (int j = 0; j < NX; ++j) ffma2(c0v, c1v, y[j], y[j], P0[j], P1[j]);
            }
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                P0[j] += (j == r0) ? T(K.wx[r0]) : T(0);
                P1[j] += (j == r1) ? T(K.wx[r1]) : T(0);
            }
        }
        // re-symmetrise (R22) through the dead Abar buffer
        if (act) {
            st_row<T, NX, true>(s.X + r0 * NX, P0);
            st_row<T, NX, true>(s.X + r1 * NX, P1);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < NX; ++j) {
            P0[j] = T(0.5) * (P0[j] + s.X[j * NX + r0]);
            P1[j] = T(0.5) * (P1[j] + s.X[j * NX + r1]);
        }
        __syncwarp();
        if (act) {
            st_row<T, NX, true>(s.P + r0 * NX, P0);
            st_row<T, NX, true>(s.P + r1 * NX, P1);
            s.p[r0] = pn0;
            s.p[r1] = pn1;
            st_row<T, NX, true>(Pp + (size_t)i * TP + r0 * NX, P0);
            st_row<T, NX, true>(Pp + (size_t)i * TP + r1 * NX, P1);
            Pp[(size_t)i * TP + NX * NX + r0] = pn0;
            Pp[(size_t)i * TP + NX * NX + r1] = pn1;
        }
        __syncwarp();
    }
    {
        const T xa = it.x0[(size_t)b * NX + r0], xc = it.x0[(size_t)b * NX + r1];
        bad = bad || !isfinite(xa) || !isfinite(xc);
    }
    // per worker: OR of bad over its 6 lanes, then lane 0 of the worker writes info
    const unsigned bm = __ballot_sync(0xffffffffu, bad && lane_act);
    const bool any_bad = ((bm >> wb) & 0x3fu) != 0u;
    if (l == 0 && act) info_out[b] = any_bad ? -1 : (fail != INT_MAX ? fail : 0);
}

// ------------------------------------------------------------------ forward + line search
// Line-search contribution of stage i (0..N+1) for every alpha slot a = 0..na (a = 0: current
// iterate, a >= 1: alpha = 2^-(a-1)): adds J_i(a) to aJ[a][lane] and ||defect_i(a)||_2 to
// aT[a][lane], the cost slope at a = 0 to g, and sets bit a of guard if the trial pitch leaves the
// Euler guard.  Tracking costs are exact quadratics in alpha (fp64); barrier arguments are
// xi0 + a dxi; the defect is (x_{i+1} - x_i) + a (dx_{i+1} - dx_i) - dt f(x_i + a dx_i, u_i + a du_i).
// Trial states and the model in F (fp32: SFU sincos / log), sums in fp64.
template <typename T>
__device__ __forceinline__ void ls_stage(const SrbdConst &K, const SrbdIter<T> &it, int b, int N, int i, int na,
                                         const T *x, const T *Dx, const T *u, const T *Du, const T *xr, const T *urf,
                                         double (*aJ)[32], double (*aT)[32], T (*sDel)[32], int lane, double &g,
                                         unsigned &guard, int a_lo = 0, int a_hi = -1, bool add_g = true) {
    // alpha slots a_lo..a_hi (default: all 0..na); add_g: this call also accumulates the slope g
    (void)sDel;
    if (a_hi < 0) a_hi = na;
    constexpr int NX = 12;
    using F = T;
    const T *xi = x + (size_t)i * NX, *dxi = Dx + (size_t)i * NX;
    const T *xri = xr + (size_t)i * NX;
    if (i == N + 1) {  // terminal cost: quadratic in alpha
        double c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            const double e = (double)xi[k] - (double)xri[k], d = (double)dxi[k];
            c0 += 0.5 * K.wxt[k] * e * e; c1 += K.wxt[k] * e * d; c2 += 0.5 * K.wxt[k] * d * d;
        }
        for (int a = a_lo; a <= a_hi; ++a) {
            const double al = a == 0 ? 0.0 : ldexp(1.0, -(a - 1));
            aJ[a][lane] += c0 + al * (c1 + al * c2);
        }
        if (add_g) g += c1;
        return;
    }
    // every row of the stage in registers with 16-byte loads (rows are 16-byte aligned)
    T xa[NX], xb1[NX], da[NX], db[NX], ua[NX], dua[NX], fe[NX];
    ld_row<T, NX, true>(xa, xi);
    ld_row<T, NX, true>(xb1, xi + NX);
    ld_row<T, NX, true>(da, dxi);
    ld_row<T, NX, true>(db, dxi + NX);
    ld_row<T, NX, true>(ua, u + (size_t)i * NX);
    ld_row<T, NX, true>(dua, Du + (size_t)i * NX);
    ld_row<T, NX, true>(fe, it.feet + ((size_t)b * (N + 1) + i) * 12);
    const uint32_t cw = *reinterpret_cast<const uint32_t *>(it.con + ((size_t)b * (N + 1) + i) * 4);
    const uint8_t cmask = (uint8_t)(((cw & 0xffu) ? 1 : 0) | ((cw & 0xff00u) ? 2 : 0) | ((cw & 0xff0000u) ? 4 : 0) |
                                    ((cw & 0xff000000u) ? 8 : 0));
    // quadratic tracking costs: c0 + c1 a + c2 a^2
    double c0 = 0, c1 = 0, c2 = 0;
    {
        T xrv[NX], urv[NX];
        ld_row<T, NX, true>(xrv, xri);
        if (urf) ld_row<T, NX, true>(urv, urf + (size_t)i * NX);
        else zero(urv);
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            const double e = (double)xa[k] - (double)xrv[k], d = (double)da[k];
            c0 += 0.5 * K.wx[k] * e * e; c1 += K.wx[k] * e * d; c2 += 0.5 * K.wx[k] * d * d;
            const double wu = ((cmask >> (k / 3)) & 1) ? K.wu_st : K.wu_sw;
            const double eu = (double)ua[k] - (double)urv[k], du_ = (double)dua[k];
            c0 += 0.5 * wu * eu * eu; c1 += wu * eu * du_; c2 += 0.5 * wu * du_ * du_;
        }
    }
    if (add_g) g += c1;
    // stance feet compacted into slots q < ns (foot (perm >> 2q) & 3); per slot the force f0 + a df.
    // Everything affine in alpha is hoisted out of the alpha loop:
    //   torque  sum_q (r_q - a dp) x (f_q + a df_q) = tau0 + a tau1 + a^2 tau2  (r_q = foothold - p),
    //   defect rows 0-2 (v) and 6-8 (F/m + g) are affine: d = A + a B.
    int ns = 0, perm = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if ((cmask >> j) & 1) { perm |= j << (2 * ns); ++ns; }
    const F dp[3] = {(F)da[0], (F)da[1], (F)da[2]};
    F f0[4][3], df[4][3];
    F tau0[3] = {F(0), F(0), F(0)}, tau1[3] = {F(0), F(0), F(0)}, tau2[3] = {F(0), F(0), F(0)};
    F Fs0[3] = {F(0), F(0), F(0)}, Fs1[3] = {F(0), F(0), F(0)};
    const F mu = (F)K.mu, fmn = (F)K.fmin, fmx = (F)K.fmax;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const bool on = q < ns;
        const int j = (perm >> (2 * q)) & 3;
        F fq[3], dq[3], rq[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // foot j's entries by compile-time selects (no runtime register indexing)
            const F uf = j == 0 ? (F)ua[c] : j == 1 ? (F)ua[3 + c] : j == 2 ? (F)ua[6 + c] : (F)ua[9 + c];
            const F df_ = j == 0 ? (F)dua[c] : j == 1 ? (F)dua[3 + c] : j == 2 ? (F)dua[6 + c] : (F)dua[9 + c];
            const F ff = j == 0 ? (F)fe[c] : j == 1 ? (F)fe[3 + c] : j == 2 ? (F)fe[6 + c] : (F)fe[9 + c];
            fq[c] = on ? uf : F(0);
            dq[c] = on ? df_ : F(0);
            rq[c] = ff - (F)xa[c];
            f0[q][c] = fq[c];
            df[q][c] = dq[c];
            Fs0[c] += fq[c];
            Fs1[c] += dq[c];
        }
        tau0[0] += rq[1] * fq[2] - rq[2] * fq[1];
        tau0[1] += rq[2] * fq[0] - rq[0] * fq[2];
        tau0[2] += rq[0] * fq[1] - rq[1] * fq[0];
        tau1[0] += (rq[1] * dq[2] - rq[2] * dq[1]) - (dp[1] * fq[2] - dp[2] * fq[1]);
        tau1[1] += (rq[2] * dq[0] - rq[0] * dq[2]) - (dp[2] * fq[0] - dp[0] * fq[2]);
        tau1[2] += (rq[0] * dq[1] - rq[1] * dq[0]) - (dp[0] * fq[1] - dp[1] * fq[0]);
        tau2[0] -= dp[1] * dq[2] - dp[2] * dq[1];
        tau2[1] -= dp[2] * dq[0] - dp[0] * dq[2];
        tau2[2] -= dp[0] * dq[1] - dp[1] * dq[0];
        if (add_g && on) {   // barrier part of the slope at a = 0
#pragma unroll
            for (int cc = 0; cc < 6; ++cc) {
                F gx, gy, gz, h;
                foot_con<F>(cc, mu, fmn, fmx, gx, gy, gz, h);
                F d1, d2;
                barrier_d12<F>(gx * fq[0] + gy * fq[1] + gz * fq[2] + h, (F)K.bmu, (F)K.bdelta, (F)K.ibd2, d1, d2);
                g += (double)d1 * (double)(gx * dq[0] + gy * dq[1] + gz * dq[2]);
            }
        }
    }
    const F dtf = (F)K.dt, im = (F)K.imass;
    // affine defect rows: 0-2 (f = v), 6-8 (f = F / m + g)
    F LA[6], LB[6];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        LA[c] = (F)(xb1[c] - xa[c]) - dtf * (F)xa[6 + c];
        LB[c] = (F)(db[c] - da[c]) - dtf * (F)da[6 + c];
        LA[3 + c] = (F)(xb1[6 + c] - xa[6 + c]) - dtf * (Fs0[c] * im + (F)K.g[c]);
        LB[3 + c] = (F)(db[6 + c] - da[6 + c]) - dtf * (Fs1[c] * im);
    }
    // nonlinear rows 3-5 (Euler rates) and 9-11 (angular acceleration): differences of the iterate / direction
    F N0[6], N1[6], th0[3], dth[3], om0[3], dom[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        N0[c] = (F)(xb1[3 + c] - xa[3 + c]);
        N1[c] = (F)(db[3 + c] - da[3 + c]);
        N0[3 + c] = (F)(xb1[9 + c] - xa[9 + c]);
        N1[3 + c] = (F)(db[9 + c] - da[9 + c]);
        th0[c] = (F)xa[3 + c]; dth[c] = (F)da[3 + c];
        om0[c] = (F)xa[9 + c]; dom[c] = (F)da[9 + c];
    }
    const F bmu = (F)K.bmu, bdl = (F)K.bdelta, ibdl = (F)K.ibd, lbd = fast_log((F)K.bdelta);
    for (int a = a_lo; a <= a_hi; ++a) {
        const double ald = a == 0 ? 0.0 : ldexp(1.0, -(a - 1));
        const F al = (F)ald;
        double J = c0 + ald * (c1 + ald * c2);
        // relaxed barriers: the logarithmic branches of a foot's six constraints
        // share one logarithm, sum_c -mu log xi_c = -mu log prod_c xi_c (xi_c >= delta > 0;
        // the product of six forces <= f_max stays far inside the fp32 range), the quadratic
        // branches are added one by one; one MUFU.LG2 per stance foot
        F Jb = F(0.);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q >= ns) break;
            const F fx = fma(al, df[q][0], f0[q][0]), fy = fma(al, df[q][1], f0[q][1]), fz = fma(al, df[q][2], f0[q][2]);
            const F mfz = mu * fz;
            const F xv[6] = {mfz - fx, mfz + fx, mfz - fy, mfz + fy, fz - fmn, fmx - fz};
            bool alllog = true;
#pragma unroll
            for (int cc = 0; cc < 6; ++cc) alllog = alllog && xv[cc] >= bdl;
            F prod = F(1.), quad = F(0.);
            if (alllog) {   // the common case: every constraint in the logarithmic branch (same product order)
#pragma unroll
                for (int cc = 0; cc < 6; ++cc) prod *= xv[cc];
            } else {
#pragma unroll
                for (int cc = 0; cc < 6; ++cc) {
                    const F t = (xv[cc] - F(2.) * bdl) * ibdl;
                    const bool lg = xv[cc] >= bdl;
                    prod *= lg ? xv[cc] : F(1.);
                    quad += lg ? F(0.) : F(0.5) * bmu * (t * t - F(1.)) - bmu * lbd;
                }
            }
            Jb += quad - bmu * fast_log(prod);
        }
        J += (double)Jb;
        F th[3], w[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) { th[c] = fma(al, dth[c], th0[c]); w[c] = fma(al, dom[c], om0[c]); }
        if (!(fabs(th[1]) < (F)kPitchGuard)) guard |= 1u << a;
        // SRBD f(x + a dx, u + a du) rows 3-5 and 9-11 (fast SFU trig): same equations as SrbdEval
        F sr, cr, sp, cp, sy, cy;
        fast_sincos(th[0], &sr, &cr);
        fast_sincos(th[1], &sp, &cp);
        fast_sincos(th[2], &sy, &cy);
        const F icp = rcp_rn(cp), tp = sp * icp;
        const F R0 = cy * cp, R1 = cy * sp * sr - sy * cr, R2 = cy * sp * cr + sy * sr;
        const F R3 = sy * cp, R4 = sy * sp * sr + cy * cr, R5 = sy * sp * cr - cy * sr;
        const F R6 = -sp, R7 = cp * sr, R8 = cp * cr;
        const F t0 = fma(al, fma(al, tau2[0], tau1[0]), tau0[0]);
        const F t1 = fma(al, fma(al, tau2[1], tau1[1]), tau0[1]);
        const F t2 = fma(al, fma(al, tau2[2], tau1[2]), tau0[2]);
        F Iw[3], rh[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) Iw[c] = (F)K.I[3 * c] * w[0] + (F)K.I[3 * c + 1] * w[1] + (F)K.I[3 * c + 2] * w[2];
        rh[0] = R0 * t0 + R3 * t1 + R6 * t2 - (w[1] * Iw[2] - w[2] * Iw[1]);
        rh[1] = R1 * t0 + R4 * t1 + R7 * t2 - (w[2] * Iw[0] - w[0] * Iw[2]);
        rh[2] = R2 * t0 + R5 * t1 + R8 * t2 - (w[0] * Iw[1] - w[1] * Iw[0]);
        F fv[6];
        fv[0] = w[0] + sr * tp * w[1] + cr * tp * w[2];
        fv[1] = cr * w[1] - sr * w[2];
        fv[2] = (sr * w[1] + cr * w[2]) * icp;
#pragma unroll
        for (int c = 0; c < 3; ++c)
            fv[3 + c] = (F)K.Iinv[3 * c] * rh[0] + (F)K.Iinv[3 * c + 1] * rh[1] + (F)K.Iinv[3 * c + 2] * rh[2];
        F d2 = F(0.);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const F dl = fma(al, LB[k], LA[k]);
            d2 = fma(dl, dl, d2);
            const F dn = fma(al, N1[k], N0[k]) - dtf * fv[k];
            d2 = fma(dn, dn, d2);
        }
        aJ[a][lane] += J;
        aT[a][lane] += (double)sqrt(d2);
    }
}

// Per-warp shared memory of k_srbd_fwd_ls: during the rollout a ring of D stage blocks
// [(Abar_i, bbar_i) | (K_i, k_i) | (P_i, p_i)] filled by cp.async D-1 stages ahead; during the line
// search the per-lane alpha partial sums (the two phases never overlap).
template <typename T>
struct FwdLsSmem {
    static constexpr int NA = 16, BLK = 3 * 156, D = sizeof(T) == 8 ? 3 : 6;
    static constexpr size_t LS = 2 * NA * 32 * sizeof(double);
    static constexpr size_t RING = (size_t)D * BLK * sizeof(T);
    static constexpr size_t PER_WARP = LS > RING ? LS : RING;
};

template <typename T, int MINB>
__global__ void __launch_bounds__(128, MINB) k_srbd_fwd_ls(SrbdConst K, SrbdIter<T> it, int B, int N, LqWork<T> ws,
                                                           T *dx, T *du, T *dlam, const int32_t *info_in, LsOut<T> so,
                                                           const int32_t *pre_info = nullptr) {
    constexpr int NX = 12, NA = 16;
    constexpr int TP = TE<NX>::SIZE;
    using KL = KE<NX, NX>;
    using SM = FwdLsSmem<T>;
    static_assert(TP == 156 && KL::SIZE == 156 && KL::K == 0, "stage block layout");
    constexpr int WPB = LsWarps<T>::value;  // warps (instances) per block
    constexpr int D = SM::D;
    __shared__ __align__(16) T sx[WPB][16];
    __shared__ __align__(16) unsigned char sraw[WPB * SM::PER_WARP];
    const int lane = threadIdx.x & 31, wl = threadIdx.x / 32;
    const int b = blockIdx.x * (blockDim.x / 32) + wl;
    if (b >= B) return;
    unsigned char *mine = sraw + (size_t)wl * SM::PER_WARP;
    const int na = K.n_alpha;
    const T *x = it.x + (size_t)b * (N + 2) * NX, *u = it.u + (size_t)b * (N + 1) * NX;
    const T *xr = it.xref + (size_t)b * (N + 2) * NX;
    const T *urf = it.uref ? it.uref + (size_t)b * (N + 1) * NX : nullptr;
    const T *x0 = it.x0 + (size_t)b * NX;
    const T *Pp = ws.Pp + (size_t)b * (N + 2) * TP;
    const T *Kk = ws.Kk + (size_t)b * (N + 1) * KL::SIZE;
    const T *Te = ws.tel + (size_t)b * (N + 1) * TP;
    T *Dx = dx + (size_t)b * (N + 2) * NX, *Du = du + (size_t)b * (N + 1) * NX, *Dl = dlam + (size_t)b * (N + 2) * NX;
    int info;
    if (info_in != nullptr) {
        info = info_in[b];
    } else {  // finalise from the pipeline's failure records (see k_finalize_info)
        const int f = ws.fail[b], pr = pre_info[b];
        info = pr != 0 ? pr : (f != kFailNone ? (f & 0xFFFFFF) : 0);
    }
    // ---------------- closed-loop rollout (one chunk of Eq. 15) and du (Eq. 6)
    T *ring = reinterpret_cast<T *>(mine);
    constexpr int CH = 156 * (int)sizeof(T) / 16;  // 16-byte chunks per 156-entry block
    constexpr int EPC = 16 / (int)sizeof(T);
    // per-lane chunk slots of a stage block, fixed for the whole rollout: chunk c = lane + 32 q of the
    // [(Abar, bbar) | (K, k) | (P, p)] block comes from array c / CH at offset (c mod CH) chunks; the
    // three arrays share the per-stage stride TP, so a stage only adds s * TP to the slot pointers
    constexpr int NQ = (3 * CH + 31) / 32;
    const T *srcq[NQ];
    int dstq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int c = lane + 32 * q;
        const int blk = c < CH ? 0 : c < 2 * CH ? 1 : 2;
        srcq[q] = (c < 3 * CH) ? (blk == 0 ? Te : blk == 1 ? Kk : Pp) + (c - blk * CH) * EPC : nullptr;
        dstq[q] = c * EPC;
    }
    auto issue = [&](int s) {  // stage s -> ring slot s % D (always commits a group)
        if (s <= N) {
            T *dst = ring + (size_t)(s % D) * SM::BLK;
            const size_t so = (size_t)s * TP;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (srcq[q]) cp_async16(dst + dstq[q], srcq[q] + so);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s0 = 0; s0 < D - 1; ++s0) issue(s0);
    const int r = lane & 15;
    const bool rowl = r < NX;
    {
        const T d0 = x0[r < NX ? r : 0] - x[r < NX ? r : 0];
        if (lane < NX) { sx[wl][r] = d0; Dx[r] = d0; }
    }
    // non-finite direction entries (dx, du, dlam) make info = -1 as on the other step paths
    // (k_finalize_info rule); checked in registers where they are produced
    bool nonfin = false;
    // lanes 0..11: dx_{i+1} = Abar_i dx_i + bbar_i (the dependent chain);
    // lanes 16..27: du_i = K_i dx_i + k_i (Eq. 6) and dlam_i = P_i dx_i + p_i (Eq. 7) off the chain
    const int roff = (lane < 16 ? 0 : 156) + (rowl ? r : 0) * NX;
    const int ooff = (lane < 16 ? 0 : 156) + NX * NX + (rowl ? r : 0);
    const int poff = 312 + (rowl ? r : 0) * NX, pbo = 312 + NX * NX + (rowl ? r : 0);
    for (int i = 0; i <= N; ++i) {
        issue(i + D - 1);
        cp_async_wait<D - 1>();
        __syncwarp();
        const T *blk = ring + (size_t)(i % D) * SM::BLK;
        T rcur[NX], xv[NX], prw[NX];
        ld_row<T, NX, true>(rcur, blk + roff);
        ld_row<T, NX, true>(xv, sx[wl]);
        const T v = row_dot<T, NX>(rcur, xv, blk[ooff]);
        T vl = T(0);
        if (lane >= 16) {
            ld_row<T, NX, true>(prw, blk + poff);
            vl = row_dot<T, NX>(prw, xv, blk[pbo]);
        }
        nonfin = nonfin || !isfinite(v) || !isfinite(vl);
        __syncwarp();
        if (rowl) {
            if (lane < 16) { sx[wl][r] = v; Dx[(size_t)(i + 1) * NX + r] = v; }
            else { Du[(size_t)i * NX + r] = v; Dl[(size_t)i * NX + r] = vl; }
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
    if (lane >= 16 && rowl) {   // dlam_{N+1} = P_{N+1} dx_{N+1} + p_{N+1}
        T prw[NX], xv[NX];
        ld_row<T, NX, true>(prw, Pp + (size_t)(N + 1) * TP + r * NX);
        ld_row<T, NX, true>(xv, sx[wl]);
        const T vl = row_dot<T, NX>(prw, xv, Pp[(size_t)(N + 1) * TP + NX * NX + r]);
        Dl[(size_t)(N + 1) * NX + r] = vl;
        nonfin = nonfin || !isfinite(vl);
    }
    if (__any_sync(0xffffffffu, nonfin) && info == 0) info = -1;
    __syncwarp();
    // ---------------- line search: lane = stage; per alpha slot a (0 = current iterate,
    // a >= 1: alpha = 2^-(a-1)); per-lane partial sums in shared memory (no unrolled alpha loop).
    // Per stage the alpha-invariant parts are computed once: the tracking costs are exact
    // quadratics c0 + c1 a + c2 a^2 (fp64), the barrier arguments are xi0 + a dxi, the defect is
    // (x_{i+1} - x_i) + a (dx_{i+1} - dx_i) - dt f(x_i + a dx_i, u_i + a du_i).  Trial states and
    // the model are evaluated in fp32 (fast sincos / log: SFU), sums in fp64.
    double(*aJ)[32] = reinterpret_cast<double(*)[32]>(mine);
    double(*aT)[32] = reinterpret_cast<double(*)[32]>(mine + NA * 32 * sizeof(double));
    T(*sDel)[32] = nullptr;
    for (int a = 0; a <= na; ++a) { aJ[a][lane] = 0.0; aT[a][lane] = 0.0; }
    unsigned guard = 0u;  // bit a: some trial state of slot a leaves the pitch guard
    double g = 0.0;
    for (int i = lane; i <= N + 1; i += 32)
        ls_stage<T>(K, it, b, N, i, na, x, Dx, u, Du, xr, urf, aJ, aT, sDel, lane, g, guard);
    // fixed-order xor butterflies: every lane ends with bitwise identical sums
    for (int a = 0; a <= na; ++a) {
        double vJ = aJ[a][lane], vT = aT[a][lane];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            vJ += __shfl_xor_sync(0xffffffffu, vJ, off);
            vT += __shfl_xor_sync(0xffffffffu, vT, off);
        }
        __syncwarp();
        aJ[a][lane] = vJ;
        aT[a][lane] = vT;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        g += __shfl_xor_sync(0xffffffffu, g, off);
        guard |= __shfl_xor_sync(0xffffffffu, guard, off);
    }
    __syncwarp();
    // initial-condition term of theta, ||xhat0 - (x0 + a dx0)||  (reading R9)
    double d0[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) d0[k] = (double)x0[k] - (double)x[k];
    const double J0 = aJ[0][lane];
    double th0;
    {
        double q = 0;
#pragma unroll
        for (int k = 0; k < NX; ++k) q += d0[k] * d0[k];
        th0 = aT[0][lane] + sqrt(q);
    }
    int jb = -1;
    double Jb = J0, thb = th0;
    if (info == 0) {
        for (int a = 1; a <= na; ++a) {
            const double al = ldexp(1.0, -(a - 1));
            double q = 0;
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                const double e = d0[k] - al * (double)Dx[k];
                q += e * e;
            }
            const double Ja = aJ[a][lane], tha = aT[a][lane] + sqrt(q);
            bool ok = !((guard >> a) & 1u) && isfinite(Ja) && isfinite(tha);
            if (ok) {
                if (th0 > K.theta_max) ok = tha <= th0;         // "reject if it further increases theta"
                else if (g < 0) ok = Ja <= J0 + K.c1 * al * g;   // Armijo on descent directions
                else ok = (Ja < J0) || (tha < th0);              // cost or theta must decrease
            }
            if (ok) { jb = a; Jb = Ja; thb = tha; break; }
        }
    }
    const T alpha = jb >= 0 ? (T)ldexp(1.0, -(jb - 1)) : T(0);
    commit_step<T>(it, so, b, N, lane, jb >= 0, alpha, J0, th0, Jb, thb, info, Dx, Du, Dl, g);
}

// ------------------------------------------- stage-parallel linearisation + element init
// One worker per (instance, stage i = 0..N+1): linearise stage i (a1) and build its value element
// (a2, Eq. 12 with S = 0, block-diagonal R^-1 in closed form; Eq. 13 for i = N+1) into
// ws.elems, plus the Eq. 4 blocks the policy needs (A, B, b, R, r) into `qp` (user layout).
template <typename T>
struct LinElemSmem {
    T B[144], F[144], Rr[144], ZB[144];
    T zr[12], c[12], pad[8];
};

template <typename T>
__global__ void __launch_bounds__(128) k_srbd_lin_elem(SrbdConst K, SrbdIter<T> it, int B, int N, LqWork<T> ws,
                                                       LqArgs<T> qp, int32_t *pre_info) {
    constexpr int WS = 16, NX = 12;
    using L = VE<NX>;
    extern __shared__ __align__(16) unsigned char smraw[];
    LinElemSmem<T> &s = reinterpret_cast<LinElemSmem<T> *>(smraw)[threadIdx.x / WS];
    const int lane = worker_lane<WS>();
    const long gw_raw = (long)blockIdx.x * (blockDim.x / WS) + threadIdx.x / WS;
    const long total = (long)B * (N + 2);
    if (__all_sync(0xffffffffu, gw_raw >= total)) return;
    const bool live = gw_raw < total;
    const long gw = live ? gw_raw : total - 1;
    const int b = (int)(gw / (N + 2)), i = (int)(gw % (N + 2));
    const int r = lane < NX ? lane : 0;
    const bool act = lane < NX, wr_g = act && live;
    const T *x = it.x + ((size_t)b * (N + 2) + i) * NX;
    const T *lam = it.lam + ((size_t)b * (N + 2) + i) * NX;
    const T *xr = it.xref + ((size_t)b * (N + 2) + i) * NX;
    T *e = ws.elems + ((size_t)b * (N + 2) + i) * L::SIZE;
    if (i == N + 1) {  // e_{N+1}: A~ = C~ = b~ = 0, P~ = W_N, p~ = W_N (x - xref) - lam  (Eq. 13)
        T z[NX], Prow[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) { z[j] = T(0); Prow[j] = (j == r) ? T(K.wxt[r]) : T(0); }
        const T pr = T(K.wxt[r]) * (x[r] - xr[r]) - lam[r];
        if (wr_g) {
            st_row<T, NX, true>(e + L::A + r * NX, z);
            st_row<T, NX, true>(e + L::C + r * NX, z);
            st_row<T, NX, true>(e + L::P + r * NX, Prow);
            e[L::b + r] = T(0);
            e[L::p + r] = pr;
            const T *xfirst = it.x + (size_t)b * (N + 2) * NX;
            const_cast<T *>(qp.dx0)[(size_t)b * NX + r] = it.x0[(size_t)b * NX + r] - xfirst[r];  // dx0 = xhat0 - x0
            if (!isfinite(x[r]) || !isfinite(lam[r]) || !isfinite(it.x0[(size_t)b * NX + r])) pre_info[b] = -1;
        }
        return;  // the partner worker of this warp only uses its own lane mask below
    }
    const size_t st = (size_t)b * (N + 1) + i;
    const T *u = it.u + st * NX, *feet = it.feet + st * 12;
    const uint8_t *con = it.con + st * 4;
    const T *ur = it.uref ? it.uref + st * NX : nullptr;
    const T *ln = lam + NX;
    const T dt = T(K.dt);
    SrbdRow<T> row;
    srbd_stage_row<T>(K, x, u, feet, con, ur, r, row, (T)it.rho_of(b));
    const bool bad = row.bad || !isfinite(lam[r]);
    const T cr = (x[r] - x[NX + r]) + dt * row.fr;  // b_i = h(x_i, u_i) - x_{i+1}
    const unsigned mask = worker_mask<WS>();
    if (act) {
        st_row<T, NX, true>(s.B + r * NX, row.Brow);
        st_row<T, NX, true>(s.F + r * NX, row.Arow);  // dt Fx
        st_row<T, NX, true>(s.Rr + r * NX, row.Rrow);
        s.c[r] = cr;
    }
    __syncwarp(mask);
    T ATl = T(0), BTl = T(0);
#pragma unroll
    for (int t = 0; t < NX; ++t) { ATl = fma(s.F[t * NX + r], ln[t], ATl); BTl = fma(s.B[t * NX + r], ln[t], BTl); }
    const T qr = T(K.wx[r]) * (x[r] - xr[r]) + ((ln[r] - lam[r]) + ATl);
    const T rr = row.rg + BTl;
    if (act) s.zr[r] = rr;
    __syncwarp(mask);
    bool fail = false;
    {   // R^-1 per foot block (closed form), z = R^-1 r, ZB = R^-1 B^T
        const int jf = r / 3, ar = r - 3 * (r / 3), o = 3 * jf;
        const T *Rb = s.Rr + o * NX + o;
        const T a00 = Rb[0], a01 = Rb[1], a02 = Rb[2];
        const T a10 = Rb[NX], a11 = Rb[NX + 1], a12 = Rb[NX + 2];
        const T a20 = Rb[2 * NX], a21 = Rb[2 * NX + 1], a22 = Rb[2 * NX + 2];
        const T c00 = a11 * a22 - a12 * a21, c01 = a02 * a21 - a01 * a22, c02 = a01 * a12 - a02 * a11;
        const T c10 = a12 * a20 - a10 * a22, c11 = a00 * a22 - a02 * a20, c12 = a02 * a10 - a00 * a12;
        const T c20 = a10 * a21 - a11 * a20, c21 = a01 * a20 - a00 * a21, c22 = a00 * a11 - a01 * a10;
        const T det = a00 * c00 + a01 * c10 + a02 * c20;
        fail = !(a00 > T(0)) || !(c22 > T(0)) || !(det > T(0)) || !isfinite(det);
        const T id = T(1) / det;
        const T q0 = (ar == 0 ? c00 : ar == 1 ? c10 : c20) * id;
        const T q1 = (ar == 0 ? c01 : ar == 1 ? c11 : c21) * id;
        const T q2 = (ar == 0 ? c02 : ar == 1 ? c12 : c22) * id;
        const T z = q0 * s.zr[o] + q1 * s.zr[o + 1] + q2 * s.zr[o + 2];
        T zb[NX];
#pragma unroll
        for (int t = 0; t < NX; ++t) zb[t] = q0 * s.B[t * NX + o] + q1 * s.B[t * NX + o + 1] + q2 * s.B[t * NX + o + 2];
        __syncwarp(mask);
        if (act) { st_row<T, NX, true>(s.ZB + r * NX, zb); s.zr[r] = z; }
    }
    __syncwarp(mask);
    T ct[NX];
    zero(ct);
    row_mat<T, NX, NX, NX>(ct, row.Brow, s.ZB);                    // C~ = B R^-1 B^T
    const T bt = cr - row_dot<T, NX>(row.Brow, s.zr, T(0));          // b~ = b - B R^-1 r
    if (wr_g) {
        T arow[NX], Prow[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) { arow[j] = (j == r ? T(1) : T(0)) + row.Arow[j]; Prow[j] = (j == r) ? T(K.wx[r]) : T(0); }
        st_row<T, NX, true>(e + L::A + r * NX, arow);
        st_row<T, NX, true>(e + L::C + r * NX, ct);
        st_row<T, NX, true>(e + L::P + r * NX, Prow);
        e[L::b + r] = bt;
        e[L::p + r] = qr;
        st_row<T, NX, true>(const_cast<T *>(qp.A) + st * NX * NX + r * NX, arow);
        st_row<T, NX, true>(const_cast<T *>(qp.Bm) + st * NX * NX + r * NX, row.Brow);
        st_row<T, NX, true>(const_cast<T *>(qp.R) + st * NX * NX + r * NX, row.Rrow);
        const_cast<T *>(qp.c)[st * NX + r] = cr;
        const_cast<T *>(qp.r)[st * NX + r] = rr;
        if (bad) pre_info[b] = -1;
        if (fail) atomicMin(ws.fail + b, i + 1);
    }
}

// ------------------------------------------------ line search for small batches (latency regime)
// grid (S, B), one warp per block and per 32 stages: every warp adds its stages' contributions per
// alpha slot, writes them to `part` ([B][S][2 NA + 2] doubles), and the last warp of an instance
// (atomic ticket) reduces the S partials in a fixed order, applies the filter rule,
// updates x, u, lam in place (Eq. 16) and writes the stats.  `cnt` ([B] ints) must be zero on
// entry and is left zero.
template <typename T>
__global__ void __launch_bounds__(32) k_srbd_ls_multi(SrbdConst K, SrbdIter<T> it, int B, int N, const T *dx,
                                                      const T *du, const T *dlam, const int32_t *info_in, LsOut<T> so,
                                                      double *part, int *cnt, int AG, const int32_t *fail = nullptr,
                                                      const int32_t *nonfin = nullptr, const int32_t *pre = nullptr) {
    // info_in == nullptr: the info word (k_finalize_info's rule) is derived here from fail / nonfin / pre
    constexpr int NX = 12, NA = 16, PW = 2 * NA + 2;
    __shared__ double aJ[NA][32], aT[NA][32];
    T(*sDel)[32] = nullptr;
    // grid (S * AG, B): block x = ag * S + sblk evaluates stages 32 sblk.. for alpha slots
    // [ag * ca, ag * ca + ca) (ca = ceil((na + 1) / AG)); slots it does not own stay zero in its partial
    const int lane = threadIdx.x, S = gridDim.x / AG, sblk = blockIdx.x % S, ag = blockIdx.x / S, b = blockIdx.y;
    const int na = K.n_alpha, ca = (na + AG) / AG;
    const int a_lo = ag * ca, a_hi = min(na, a_lo + ca - 1);
    const T *x = it.x + (size_t)b * (N + 2) * NX, *u = it.u + (size_t)b * (N + 1) * NX;
    const T *xr = it.xref + (size_t)b * (N + 2) * NX;
    const T *urf = it.uref ? it.uref + (size_t)b * (N + 1) * NX : nullptr;
    const T *Dx = dx + (size_t)b * (N + 2) * NX, *Du = du + (size_t)b * (N + 1) * NX;
    for (int a = 0; a <= na; ++a) { aJ[a][lane] = 0.0; aT[a][lane] = 0.0; }
    double g = 0.0;
    unsigned guard = 0u;
    const int i = sblk * 32 + lane;
    if (i <= N + 1 && a_lo <= a_hi)
        ls_stage<T>(K, it, b, N, i, na, x, Dx, u, Du, xr, urf, aJ, aT, sDel, lane, g, guard, a_lo, a_hi, ag == 0);
    __syncwarp();
    const int SG = S * AG;
    double *pw = part + ((size_t)b * SG + blockIdx.x) * PW;
    for (int a = 0; a <= na; ++a) {
        double vJ = aJ[a][lane], vT = aT[a][lane];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            vJ += __shfl_xor_sync(0xffffffffu, vJ, off);
            vT += __shfl_xor_sync(0xffffffffu, vT, off);
        }
        if (lane == 0) { pw[a] = vJ; pw[NA + a] = vT; }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        g += __shfl_xor_sync(0xffffffffu, g, off);
        guard |= __shfl_xor_sync(0xffffffffu, guard, off);
    }
    if (lane == 0) { pw[2 * NA] = g; pw[2 * NA + 1] = (double)guard; }
    __threadfence();
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(cnt + b, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket != SG - 1) return;
    __threadfence();
    // last warp of instance b: fixed-order reduction over the S stage partials of each alpha slot's
    // own group (lane a <= na reads group a / ca; the slope g comes from group 0), L2 loads after
    // the fence: the same sums in the same order as with one group
    const double *pb = part + (size_t)b * SG * PW;
    const double *pg = pb + (size_t)(lane <= na ? lane / ca : 0) * S * PW;
    double J = 0.0, th = 0.0, gg = 0.0;
    unsigned gd = 0u;
    for (int t = 0; t < S; ++t) {
        if (lane <= na) {
            J += __ldcg(pg + (size_t)t * PW + lane);
            th += __ldcg(pg + (size_t)t * PW + NA + lane);
            gd |= (unsigned)__ldcg(pg + (size_t)t * PW + 2 * NA + 1);
        }
        gg += __ldcg(pb + (size_t)t * PW + 2 * NA);
    }
    const T *x0 = it.x0 + (size_t)b * NX;
    const double al = lane == 0 ? 0.0 : ldexp(1.0, -(lane - 1));
    {
        double q = 0;
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            const double e = ((double)x0[k] - (double)x[k]) - al * (double)Dx[k];
            q += e * e;
        }
        th += sqrt(q);
    }
    const double J0 = __shfl_sync(0xffffffffu, J, 0), th0 = __shfl_sync(0xffffffffu, th, 0);
    int info;
    if (info_in != nullptr) {
        info = info_in[b];
    } else {
        info = fail[b] != kFailNone ? (fail[b] & 0xFFFFFF) : (nonfin[b] ? -1 : 0);
        if (pre != nullptr && pre[b] != 0) info = pre[b];
    }
    bool ok = false;
    if (lane >= 1 && lane <= na && info == 0) {
        ok = !((gd >> lane) & 1u) && isfinite(J) && isfinite(th);
        if (ok) {
            if (th0 > K.theta_max) ok = th <= th0;
            else if (gg < 0) ok = J <= J0 + K.c1 * al * gg;
            else ok = (J < J0) || (th < th0);
        }
    }
    const unsigned acc = __ballot_sync(0xffffffffu, ok);
    const int jb = acc ? __ffs(acc) - 1 : 0;
    const double Jb = __shfl_sync(0xffffffffu, J, jb), thb = __shfl_sync(0xffffffffu, th, jb);
    const T alpha = acc ? (T)ldexp(1.0, -(jb - 1)) : T(0);
    commit_step<T>(it, so, b, N, lane, acc != 0u, alpha, J0, th0, Jb, thb, info, Dx, Du, dlam + (size_t)b * (N + 2) * NX, gg);
    if (lane == 0) cnt[b] = 0;
}

// ------------------------------------------------------------- closed loop (NEXT-1)
// Warm start of the next tick: x_i <- x_{i+1}, u_i <- u_{i+1}, lam_i <- lam_{i+1}; last entries kept.
// One thread per (instance, array, component) walks the stages in ascending order (in place).
template <typename T>
__global__ void k_srbd_shift(SrbdIter<T> it, int B, int N) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)B * 36) return;
    const int b = (int)(t / 36), a = (int)(t % 36) / 12, k = (int)(t % 12);
    T *base = a == 0 ? const_cast<T *>(it.x) + (size_t)b * (N + 2) * 12
            : a == 1 ? const_cast<T *>(it.u) + (size_t)b * (N + 1) * 12
                     : const_cast<T *>(it.lam) + (size_t)b * (N + 2) * 12;
    const int len = a == 1 ? N + 1 : N + 2;
    for (int i = 0; i + 1 < len; ++i) base[(size_t)i * 12 + k] = base[(size_t)(i + 1) * 12 + k];
}

// Batched SRBD plant: classical RK4 of the continuous dynamics (same model as the MPC), `sub`
// substeps over dt, zero-order-hold input u_hold, stage-0 contacts / footholds, optional external
// world force on the CoM.  One thread per instance.
template <typename T>
__global__ void k_srbd_plant(SrbdConst K, SrbdIter<T> it, int B, int N, T *xp, const T *uh, const T *ext, T dt, int sub) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    T x[12], u[12], fe[12];
    uint8_t con[4];
#pragma unroll
    for (int k = 0; k < 12; ++k) { x[k] = xp[(size_t)b * 12 + k]; u[k] = uh[(size_t)b * 12 + k]; fe[k] = it.feet[(size_t)b * (N + 1) * 12 + k]; }
#pragma unroll
    for (int j = 0; j < 4; ++j) con[j] = it.con[(size_t)b * (N + 1) * 4 + j];
    T Fe[3] = {T(0), T(0), T(0)};
    if (ext) for (int c = 0; c < 3; ++c) Fe[c] = ext[(size_t)b * 3 + c];
    auto f = [&](const T *xs, T *out) {
        SrbdEval<T> ev;
        ev.init(K, xs, u, fe, con);
#pragma unroll
        for (int k = 0; k < 12; ++k) out[k] = ev.f(K, xs, k);
        for (int c = 0; c < 3; ++c) out[6 + c] += Fe[c] / T(K.mass);
    };
    const T h = dt / T(sub);
    for (int s = 0; s < sub; ++s) {
        T k1[12], k2[12], k3[12], k4[12], y[12];
        f(x, k1);
#pragma unroll
        for (int k = 0; k < 12; ++k) y[k] = x[k] + T(0.5) * h * k1[k];
        f(y, k2);
#pragma unroll
        for (int k = 0; k < 12; ++k) y[k] = x[k] + T(0.5) * h * k2[k];
        f(y, k3);
#pragma unroll
        for (int k = 0; k < 12; ++k) y[k] = x[k] + h * k3[k];
        f(y, k4);
#pragma unroll
        for (int k = 0; k < 12; ++k) x[k] += h / T(6) * (k1[k] + T(2) * k2[k] + T(2) * k3[k] + k4[k]);
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) xp[(size_t)b * 12 + k] = x[k];
}

}  // namespace pdilqr
