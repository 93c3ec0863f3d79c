// adjoint.cuh -- adjoint of the LQ solve (NEXT-4, include/pdilqr.h pdilqr_solve_lq_adjoint).
// The KKT matrix M of Eq. 4 is symmetric, so dL/drhs = w with M w = g: the backward pass is one
// more run of the same parallel scans (element init, reverse scan, policy, forward scan, dual
// update) with the linear terms built from the upstream gradient g (k_adj_rhs), followed by the
// rank-1 outer products dL/dM = -w z^T per stage block (k_adj_grad).  Both kernels are HBM-bound
// elementwise passes over [B][N+1] stage blocks.
#pragma once
#include "lq.cuh"

namespace pdilqr {

template <typename T>
struct AdjRhs {       // linear terms of the adjoint LQ (workspace), layouts as pdilqr_lq
    T *q, *r, *c, *pt, *dx0;
};

template <typename T>
struct AdjIn {        // forward solution z and adjoint solution w (device)
    const T *dx, *du, *dl, *wx, *wu, *wl;
};

template <typename T>
struct AdjGrad {      // user gradient buffers, layouts as pdilqr_lq (any may be null)
    T *A, *Bm, *c, *Q, *R, *S, *q, *r, *Pt, *pt, *dx0;
};

// q'_i = -g_dx[i] (i <= N), p'_{N+1} = -g_dx[N+1], r'_i = -g_du[i], dx0' = -g_dlam[0],
// c'_i = -g_dlam[i+1]; a null gradient array contributes zeros.  One thread per element.
template <typename T>
__global__ void __launch_bounds__(256) k_adj_rhs(int B, int N, int n, int m, const T *gdx, const T *gdu,
                                                 const T *gdl, AdjRhs<T> o) {
    const long nx = (long)(N + 2) * n, nu = (long)(N + 1) * m;
    const long per = nx + nu + nx;
    const long tot = (long)B * per;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < tot; t += (long)gridDim.x * blockDim.x) {
        const long b = t / per, e = t - b * per;
        if (e < nx) {                              // from g_dx: q (stages 0..N), p_term (node N+1)
            const T v = gdx ? -gdx[b * nx + e] : T(0);
            const long i = e / n, k = e - i * n;
            if (i <= N) o.q[(b * (N + 1) + i) * n + k] = v;
            else o.pt[b * n + k] = v;
        } else if (e < nx + nu) {                  // from g_du: r
            const long f = e - nx;
            o.r[b * nu + f] = gdu ? -gdu[b * nu + f] : T(0);
        } else {                                   // from g_dlam: dx0 (node 0), c (nodes 1..N+1)
            const long f = e - nx - nu;
            const T v = gdl ? -gdl[b * nx + f] : T(0);
            const long i = f / n, k = f - i * n;
            if (i == 0) o.dx0[b * n + k] = v;
            else o.c[(b * (N + 1) + (i - 1)) * n + k] = v;
        }
    }
}

// Outer products of one stage block per thread-strided element: for stage i of instance b,
// gQ = -wx dx^T, gR = -wu du^T, gS = -(wu dx^T + du wx^T), gA = -(wl' dx^T + dl' wx^T),
// gB = -(wl' du^T + dl' wu^T) with ' = node i+1, and the vector gradients; node N+1 gives gPt, gpt.
template <typename T>
__global__ void __launch_bounds__(256) k_adj_grad(int B, int N, int n, int m, AdjIn<T> z, AdjGrad<T> g) {
    const long nn = (long)n * n, mm = (long)m * m, nm = (long)n * m;
    // per instance: N+1 stages x (2 nn [A, Q] + nm [B] + mm [R] + nm [S] + n [q] + m [r] + n [c]),
    // then the terminal nn [Pt] + n [pt] + n [dx0]
    const long ps = 2 * nn + 2 * nm + mm + 2 * n + m;
    const long per = (long)(N + 1) * ps + nn + 2 * n;
    const long tot = (long)B * per;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < tot; t += (long)gridDim.x * blockDim.x) {
        const long b = t / per;
        long e = t - b * per;
        const T *dx = z.dx + b * (N + 2) * n, *wx = z.wx + b * (N + 2) * n;
        const T *dl = z.dl + b * (N + 2) * n, *wl = z.wl + b * (N + 2) * n;
        const T *du = z.du + b * (N + 1) * m, *wu = z.wu + b * (N + 1) * m;
        if (e < (N + 1) * ps) {
            const long i = e / ps;
            e -= i * ps;
            const T *xi = dx + i * n, *wxi = wx + i * n, *ui = du + i * m, *wui = wu + i * m;
            const T *l1 = dl + (i + 1) * n, *wl1 = wl + (i + 1) * n;
            const long sb = b * (N + 1) + i;
            if (e < nn) {                                  // A_i (n x n): row r, col c
                const long r = e / n, c = e - r * n;
                if (g.A) g.A[sb * nn + e] = -(wl1[r] * xi[c] + l1[r] * wxi[c]);
            } else if ((e -= nn) < nn) {                   // Q_i
                const long r = e / n, c = e - r * n;
                if (g.Q) g.Q[sb * nn + e] = -wxi[r] * xi[c];
            } else if ((e -= nn) < nm) {                   // B_i (n x m)
                const long r = e / m, c = e - r * m;
                if (g.Bm) g.Bm[sb * nm + e] = -(wl1[r] * ui[c] + l1[r] * wui[c]);
            } else if ((e -= nm) < mm) {                   // R_i
                const long r = e / m, c = e - r * m;
                if (g.R) g.R[sb * mm + e] = -wui[r] * ui[c];
            } else if ((e -= mm) < nm) {                   // S_i (m x n)
                const long r = e / n, c = e - r * n;
                if (g.S) g.S[sb * nm + e] = -(wui[r] * xi[c] + ui[r] * wxi[c]);
            } else if ((e -= nm) < n) {                    // q_i
                if (g.q) g.q[sb * n + e] = -wxi[e];
            } else if ((e -= n) < m) {                     // r_i
                if (g.r) g.r[sb * m + e] = -wui[e];
            } else {                                       // c_i
                e -= m;
                if (g.c) g.c[sb * n + e] = -wl1[e];
            }
        } else {
            e -= (N + 1) * ps;
            const T *xt = dx + (N + 1) * n, *wxt = wx + (N + 1) * n;
            if (e < nn) {
                const long r = e / n, c = e - r * n;
                if (g.Pt) g.Pt[b * nn + e] = -wxt[r] * xt[c];
            } else if ((e -= nn) < n) {
                if (g.pt) g.pt[b * n + e] = -wxt[e];
            } else {
                e -= n;
                if (g.dx0) g.dx0[b * n + e] = -wl[e];
            }
        }
    }
}

}  // namespace pdilqr
