/*
 * oracle/pdilqr_oracle.c -- plain fp64 CPU oracle for the Primal-Dual iLQR hot path
 * (arXiv 2506.07823, /root/reference/PAPER.md; cited as P:<line>).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may load this file.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs call it.  It shares no code, header, table or helper with the CUDA path
 * (paper_2506_07823_b200/csrc); the two are written independently from the paper.
 *
 * What it computes, and how:
 *  - LQ/KKT subproblem (Eq. 4): the unique KKT solution, obtained by the
 *    sequential Riccati recursion (Eq. 5), the forward pass (Eq. 6)
 *    and the dual update (Eq. 7).  No scan, no blocking, no reordering.
 *  - SRBD model with ZYX Euler angles (n=12, reading R13),
 *    explicit Euler discretisation (reading R14), analytic Jacobians.
 *  - Gauss-Newton cost + relaxed barriers, Lagrangian gradients q,r.
 *  - Filter line search on the fixed grid alpha in {2^0..2^-9}, linear
 *    update (Eq. 16), constraint violation theta (Eq. 17, reading R9).
 *
 * Parity pins for every function live in tests/test_oracle_*.py.
 *
 * Array conventions (one instance, row-major, fp64):
 *   A[N+1][n][n] Bm[N+1][n][m] c[N+1][n] Q[N+1][n][n] R[N+1][m][m] S[N+1][m][n]
 *   q[N+1][n] r[N+1][m] Pt[n][n] pt[n] dx0[n]
 *   K[N+1][m][n] k[N+1][m] P[N+2][n][n] p[N+2][n]
 *   dx[N+2][n] du[N+1][m] dlam[N+2][n]
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX2(i, j, ld) ((size_t)(i) * (size_t)(ld) + (size_t)(j))

/* ------------------------------------------------------------------------- */
/* small dense helpers (plain loops)                                         */
/* ------------------------------------------------------------------------- */

/* Cholesky G = L L^T in place (lower triangle).  Returns 0 on success, 1 if G is
 * not (numerically) positive definite. */
static int chol(int m, double *G) {
    for (int j = 0; j < m; ++j) {
        double d = G[IDX2(j, j, m)];
        for (int k = 0; k < j; ++k) d -= G[IDX2(j, k, m)] * G[IDX2(j, k, m)];
        if (!(d > 0.0)) return 1;
        d = sqrt(d);
        G[IDX2(j, j, m)] = d;
        for (int i = j + 1; i < m; ++i) {
            double s = G[IDX2(i, j, m)];
            for (int k = 0; k < j; ++k) s -= G[IDX2(i, k, m)] * G[IDX2(j, k, m)];
            G[IDX2(i, j, m)] = s / d;
        }
    }
    return 0;
}

/* Solve (L L^T) X = Y for X in place; Y is m x ncol row-major. */
static void chol_solve(int m, const double *L, int ncol, double *Y) {
    for (int c = 0; c < ncol; ++c) {
        for (int i = 0; i < m; ++i) { /* forward: L z = y */
            double s = Y[IDX2(i, c, ncol)];
            for (int k = 0; k < i; ++k) s -= L[IDX2(i, k, m)] * Y[IDX2(k, c, ncol)];
            Y[IDX2(i, c, ncol)] = s / L[IDX2(i, i, m)];
        }
        for (int i = m - 1; i >= 0; --i) { /* backward: L^T x = z */
            double s = Y[IDX2(i, c, ncol)];
            for (int k = i + 1; k < m; ++k) s -= L[IDX2(k, i, m)] * Y[IDX2(k, c, ncol)];
            Y[IDX2(i, c, ncol)] = s / L[IDX2(i, i, m)];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* LQ subproblem: Riccati (Eq. 5), rollout (Eq. 6), dual update (Eq. 7)     */
/* ------------------------------------------------------------------------- */

/* Eq. 5, for i = N..0, starting from P_{N+1} = Pt, p_{N+1} = pt:
 *   G = R + B^T P' B,  H = S + B^T P' A,  h = B^T (p' + P' b) + r,
 *   K = -G^{-1} H,     k = -G^{-1} h,
 *   P = Q + A^T P' A + K^T H,   p = q + A^T (p' + P' b) + K^T h,
 * with P re-symmetrised after each step (exact-arithmetic identity).
 * Returns 0, or 1 + i if G_i is not positive definite (SPEC S:45 names the node). */
int oracle_riccati(int N, int n, int m,
                   const double *A, const double *Bm, const double *c,
                   const double *Q, const double *R, const double *S,
                   const double *q, const double *r,
                   const double *Pt, const double *pt,
                   double *K, double *k, double *P, double *p) {
    const size_t nn = (size_t)n * n, nm = (size_t)n * m, mm = (size_t)m * m;
    double *PB = malloc(sizeof(double) * nm);      /* P' B      (n x m) */
    double *PA = malloc(sizeof(double) * nn);      /* P' A      (n x n) */
    double *G = malloc(sizeof(double) * mm);
    double *Y = malloc(sizeof(double) * (size_t)m * (n + 1)); /* [H | h] -> G^-1 [H | h] */
    double *Hh = malloc(sizeof(double) * (size_t)m * (n + 1)); /* copy of [H | h] */
    double *w = malloc(sizeof(double) * n);        /* p' + P' b */
    int status = 0;

    memcpy(P + (size_t)(N + 1) * nn, Pt, sizeof(double) * nn);
    memcpy(p + (size_t)(N + 1) * n, pt, sizeof(double) * n);

    for (int i = N; i >= 0; --i) {
        const double *Ai = A + (size_t)i * nn, *Bi = Bm + (size_t)i * nm, *bi = c + (size_t)i * n;
        const double *Qi = Q + (size_t)i * nn, *Ri = R + (size_t)i * mm, *Si = S + (size_t)i * nm;
        const double *qi = q + (size_t)i * n, *ri = r + (size_t)i * m;
        const double *Pn = P + (size_t)(i + 1) * nn, *pn = p + (size_t)(i + 1) * n;
        double *Pi = P + (size_t)i * nn, *pi = p + (size_t)i * n;
        double *Ki = K + (size_t)i * nm, *ki = k + (size_t)i * m;

        for (int a = 0; a < n; ++a)
            for (int b = 0; b < m; ++b) {
                double s = 0;
                for (int t = 0; t < n; ++t) s += Pn[IDX2(a, t, n)] * Bi[IDX2(t, b, m)];
                PB[IDX2(a, b, m)] = s;
            }
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                double s = 0;
                for (int t = 0; t < n; ++t) s += Pn[IDX2(a, t, n)] * Ai[IDX2(t, b, n)];
                PA[IDX2(a, b, n)] = s;
            }
        for (int a = 0; a < n; ++a) {
            double s = pn[a];
            for (int t = 0; t < n; ++t) s += Pn[IDX2(a, t, n)] * bi[t];
            w[a] = s;
        }
        /* G = R + B^T P' B */
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) {
                double s = Ri[IDX2(a, b, m)];
                for (int t = 0; t < n; ++t) s += Bi[IDX2(t, a, m)] * PB[IDX2(t, b, m)];
                G[IDX2(a, b, m)] = s;
            }
        /* H = S + B^T P' A  -> Y[:, 0:n];  h = B^T w + r -> Y[:, n] */
        for (int a = 0; a < m; ++a) {
            for (int b = 0; b < n; ++b) {
                double s = Si[IDX2(a, b, n)];
                for (int t = 0; t < n; ++t) s += Bi[IDX2(t, a, m)] * PA[IDX2(t, b, n)];
                Y[IDX2(a, b, n + 1)] = s;
            }
            double s = ri[a];
            for (int t = 0; t < n; ++t) s += Bi[IDX2(t, a, m)] * w[t];
            Y[IDX2(a, n, n + 1)] = s;
        }
        /* P_i = Q + A^T P' A + K^T H, p_i = q + A^T w + K^T h */
        memcpy(Hh, Y, sizeof(double) * (size_t)m * (n + 1));
        if (chol(m, G)) { status = 1 + i; break; }
        chol_solve(m, G, n + 1, Y); /* Y = G^{-1} [H | h] */
        for (int a = 0; a < m; ++a) {
            for (int b = 0; b < n; ++b) Ki[IDX2(a, b, n)] = -Y[IDX2(a, b, n + 1)];
            ki[a] = -Y[IDX2(a, n, n + 1)];
        }
        for (int a = 0; a < n; ++a) {
            for (int b = 0; b < n; ++b) {
                double s = Qi[IDX2(a, b, n)];
                for (int t = 0; t < n; ++t) s += Ai[IDX2(t, a, n)] * PA[IDX2(t, b, n)];
                for (int t = 0; t < m; ++t) s += Ki[IDX2(t, a, n)] * Hh[IDX2(t, b, n + 1)];
                Pi[IDX2(a, b, n)] = s;
            }
            double s = qi[a];
            for (int t = 0; t < n; ++t) s += Ai[IDX2(t, a, n)] * w[t];
            for (int t = 0; t < m; ++t) s += Ki[IDX2(t, a, n)] * Hh[IDX2(t, n, n + 1)];
            pi[a] = s;
        }
        /* P_i is symmetric in exact arithmetic; re-symmetrise it (DESIGN.md reading
         * R22) so that rounding asymmetry cannot accumulate over long horizons. */
        for (int a = 0; a < n; ++a)
            for (int b = a + 1; b < n; ++b) {
                double v = 0.5 * (Pi[IDX2(a, b, n)] + Pi[IDX2(b, a, n)]);
                Pi[IDX2(a, b, n)] = v;
                Pi[IDX2(b, a, n)] = v;
            }
    }
    free(PB); free(PA); free(G); free(Y); free(Hh); free(w);
    return status;
}

/* Eq. 6: du_i = K_i dx_i + k_i ; dx_{i+1} = A_i dx_i + B_i du_i + b_i,
 * dx_0 = xhat_0 - x_0.  Eq. 7: dlam_i = P_i dx_i + p_i, i=0..N+1. */
void oracle_rollout_dual(int N, int n, int m,
                         const double *A, const double *Bm, const double *c,
                         const double *K, const double *k,
                         const double *P, const double *p, const double *dx0,
                         double *dx, double *du, double *dlam) {
    const size_t nn = (size_t)n * n, nm = (size_t)n * m;
    memcpy(dx, dx0, sizeof(double) * n);
    for (int i = 0; i <= N; ++i) {
        const double *xi = dx + (size_t)i * n;
        double *ui = du + (size_t)i * m;
        double *xn = dx + (size_t)(i + 1) * n;
        for (int a = 0; a < m; ++a) {
            double s = k[(size_t)i * m + a];
            for (int t = 0; t < n; ++t) s += K[(size_t)i * nm + IDX2(a, t, n)] * xi[t];
            ui[a] = s;
        }
        for (int a = 0; a < n; ++a) {
            double s = c[(size_t)i * n + a];
            for (int t = 0; t < n; ++t) s += A[(size_t)i * nn + IDX2(a, t, n)] * xi[t];
            for (int t = 0; t < m; ++t) s += Bm[(size_t)i * nm + IDX2(a, t, m)] * ui[t];
            xn[a] = s;
        }
    }
    for (int i = 0; i <= N + 1; ++i)
        for (int a = 0; a < n; ++a) {
            double s = p[(size_t)i * n + a];
            for (int t = 0; t < n; ++t) s += P[(size_t)i * nn + IDX2(a, t, n)] * dx[(size_t)i * n + t];
            dlam[(size_t)i * n + a] = s;
        }
}

/* The whole LQ solve for one instance.  K,k,P,p may be NULL (then scratch is used). */
int oracle_solve_lq(int N, int n, int m,
                    const double *A, const double *Bm, const double *c,
                    const double *Q, const double *R, const double *S,
                    const double *q, const double *r,
                    const double *Pt, const double *pt, const double *dx0,
                    double *dx, double *du, double *dlam,
                    double *K, double *k, double *P, double *p) {
    const size_t nn = (size_t)n * n, nm = (size_t)n * m;
    double *Kw = K ? K : malloc(sizeof(double) * (N + 1) * nm);
    double *kw = k ? k : malloc(sizeof(double) * (N + 1) * m);
    double *Pw = P ? P : malloc(sizeof(double) * (N + 2) * nn);
    double *pw = p ? p : malloc(sizeof(double) * (N + 2) * n);
    int st = oracle_riccati(N, n, m, A, Bm, c, Q, R, S, q, r, Pt, pt, Kw, kw, Pw, pw);
    if (st == 0) oracle_rollout_dual(N, n, m, A, Bm, c, Kw, kw, Pw, pw, dx0, dx, du, dlam);
    if (!K) free(Kw);
    if (!k) free(kw);
    if (!P) free(Pw);
    if (!p) free(pw);
    return st;
}

/* Adjoint of the LQ solve (NEXT-4; the differentiable solver of P:61-62): z = (dx, du, dlam)
 * solves the symmetric KKT system M z = rhs of Eq. 4, so for a loss L with dL/dz = g,
 *   w = M^{-1} g,  dL/drhs = w,  dL/dM = -w z^T   (dL = w^T (d rhs - dM z)).
 * M w = g is itself an LQ problem with the same matrices and the linear terms
 *   q'_i = -g_dx[i] (i <= N), r'_i = -g_du[i], p'_{N+1} = -g_dx[N+1], dx0' = -g_dlam[0],
 *   c'_i = -g_dlam[i+1],
 * solved here by the same sequential Riccati recursion (oracle_solve_lq).  Then, block by block of
 * M (Q_i, R_i, S_i / S_i^T, P_{N+1}, and the constraint Jacobian blocks A_i / A_i^T, B_i / B_i^T):
 *   gQ_i = -w_dx[i] dx[i]^T, gR_i = -w_du[i] du[i]^T, gS_i = -(w_du[i] dx[i]^T + du[i] w_dx[i]^T),
 *   gP_{N+1} = -w_dx[N+1] dx[N+1]^T, gA_i = -(w_dlam[i+1] dx[i]^T + dlam[i+1] w_dx[i]^T),
 *   gB_i = -(w_dlam[i+1] du[i]^T + dlam[i+1] w_du[i]^T);
 * and from rhs = -(q, r, p_{N+1}; dx0, c): gq_i = -w_dx[i], gr_i = -w_du[i], gp_{N+1} = -w_dx[N+1],
 * gdx0 = -w_dlam[0], gc_i = -w_dlam[i+1].  Returns the solve's status. */
int oracle_solve_lq_adjoint(int N, int n, int m,
                            const double *A, const double *Bm, const double *Q, const double *R,
                            const double *S, const double *Pt,
                            const double *dx, const double *du, const double *dlam,
                            const double *gdx, const double *gdu, const double *gdlam,
                            double *gA, double *gB, double *gc, double *gQ, double *gR, double *gS,
                            double *gq, double *gr, double *gPt, double *gpt, double *gdx0) {
    const size_t S1 = (size_t)(N + 1), nn = (size_t)n * n, nm = (size_t)n * m, mm = (size_t)m * m;
    double *q2 = malloc(sizeof(double) * S1 * n), *r2 = malloc(sizeof(double) * S1 * m);
    double *c2 = malloc(sizeof(double) * S1 * n), *pt2 = malloc(sizeof(double) * n);
    double *d02 = malloc(sizeof(double) * n);
    double *wx = malloc(sizeof(double) * (S1 + 1) * n), *wu = malloc(sizeof(double) * S1 * m);
    double *wl = malloc(sizeof(double) * (S1 + 1) * n);
    for (size_t i = 0; i <= (size_t)N; ++i) {
        for (int a = 0; a < n; ++a) q2[i * n + a] = -gdx[i * n + a];
        for (int a = 0; a < m; ++a) r2[i * m + a] = -gdu[i * m + a];
        for (int a = 0; a < n; ++a) c2[i * n + a] = -gdlam[(i + 1) * n + a];
    }
    for (int a = 0; a < n; ++a) { pt2[a] = -gdx[(S1) * n + a]; d02[a] = -gdlam[a]; }
    int st = oracle_solve_lq(N, n, m, A, Bm, c2, Q, R, S, q2, r2, Pt, pt2, d02, wx, wu, wl,
                             NULL, NULL, NULL, NULL);
    if (st == 0) {
        for (size_t i = 0; i <= (size_t)N; ++i) {
            const double *xi = dx + i * n, *wxi = wx + i * n, *ui = du + i * m, *wui = wu + i * m;
            const double *l1 = dlam + (i + 1) * n, *wl1 = wl + (i + 1) * n;
            for (int a = 0; a < n; ++a)
                for (int b = 0; b < n; ++b) {
                    gQ[i * nn + IDX2(a, b, n)] = -wxi[a] * xi[b];
                    gA[i * nn + IDX2(a, b, n)] = -(wl1[a] * xi[b] + l1[a] * wxi[b]);
                }
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b) gR[i * mm + IDX2(a, b, m)] = -wui[a] * ui[b];
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < n; ++b) gS[i * nm + IDX2(a, b, n)] = -(wui[a] * xi[b] + ui[a] * wxi[b]);
            for (int a = 0; a < n; ++a)
                for (int b = 0; b < m; ++b) gB[i * nm + IDX2(a, b, m)] = -(wl1[a] * ui[b] + l1[a] * wui[b]);
            for (int a = 0; a < n; ++a) { gq[i * n + a] = -wxi[a]; gc[i * n + a] = -wl1[a]; }
            for (int a = 0; a < m; ++a) gr[i * m + a] = -wui[a];
        }
        const double *xt = dx + S1 * n, *wxt = wx + S1 * n;
        for (int a = 0; a < n; ++a) {
            for (int b = 0; b < n; ++b) gPt[IDX2(a, b, n)] = -wxt[a] * xt[b];
            gpt[a] = -wxt[a];
            gdx0[a] = -wl[a];
        }
    }
    free(q2); free(r2); free(c2); free(pt2); free(d02); free(wx); free(wu); free(wl);
    return st;
}

/* Batched LQ solve over B independent instances (batch-outermost arrays). */
void oracle_solve_lq_batch(int Bn, int N, int n, int m,
                           const double *A, const double *Bm, const double *c,
                           const double *Q, const double *R, const double *S,
                           const double *q, const double *r,
                           const double *Pt, const double *pt, const double *dx0,
                           double *dx, double *du, double *dlam, int32_t *info, int nthreads) {
    const size_t nn = (size_t)n * n, nm = (size_t)n * m, mm = (size_t)m * m;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int b = 0; b < Bn; ++b) {
        const size_t S1 = (size_t)(N + 1);
        info[b] = oracle_solve_lq(N, n, m, A + b * S1 * nn, Bm + b * S1 * nm, c + b * S1 * n,
                                  Q + b * S1 * nn, R + b * S1 * mm, S + b * S1 * nm,
                                  q + b * S1 * n, r + b * S1 * m, Pt + b * nn, pt + b * n,
                                  dx0 + b * (size_t)n, dx + b * (S1 + 1) * n, du + b * S1 * m,
                                  dlam + b * (S1 + 1) * n, NULL, NULL, NULL, NULL);
    }
}

/* ------------------------------------------------------------------------- */
/* SRBD model, ZYX Euler angles (reading R13), explicit Euler    */
/* ------------------------------------------------------------------------- */
/* state x = [p(3) world position, Theta(3) = (roll, pitch, yaw), v(3) world velocity,
 *            w(3) body angular velocity];  input u = [f_0 .. f_3] world-frame GRFs.    */

typedef struct {
    double dt, mass, inertia[9], gravity[3];
    double w_x[12], w_x_term[12], w_u_stance, w_u_swing;
    double mu_friction, f_min, f_max, barrier_mu, barrier_delta;
} oracle_srbd_params;

#define NX 12
#define NU 12
#define NFEET 4
#define PITCH_GUARD (M_PI / 2.0 - 0.1)

static void mat3_mul(const double *X, const double *Y, double *Z) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int t = 0; t < 3; ++t) s += X[3 * i + t] * Y[3 * t + j];
            Z[3 * i + j] = s;
        }
}

/* inverse of a 3x3 matrix by the adjugate formula */
static void mat3_inv(const double *M, double *Mi) {
    double a = M[0], b = M[1], c = M[2], d = M[3], e = M[4], f = M[5], g = M[6], h = M[7], i = M[8];
    double det = a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
    Mi[0] = (e * i - f * h) / det; Mi[1] = (c * h - b * i) / det; Mi[2] = (b * f - c * e) / det;
    Mi[3] = (f * g - d * i) / det; Mi[4] = (a * i - c * g) / det; Mi[5] = (c * d - a * f) / det;
    Mi[6] = (d * h - e * g) / det; Mi[7] = (b * g - a * h) / det; Mi[8] = (a * e - b * d) / det;
}

/* R(Theta) = Rz(yaw) Ry(pitch) Rx(roll) and its three partial derivatives. */
static void rot_zyx(const double *th, double *R, double *dR /* [3][9] or NULL */) {
    double cr = cos(th[0]), sr = sin(th[0]), cp = cos(th[1]), sp = sin(th[1]);
    double cy = cos(th[2]), sy = sin(th[2]);
    double Rx[9] = {1, 0, 0, 0, cr, -sr, 0, sr, cr};
    double Ry[9] = {cp, 0, sp, 0, 1, 0, -sp, 0, cp};
    double Rz[9] = {cy, -sy, 0, sy, cy, 0, 0, 0, 1};
    double T[9];
    mat3_mul(Ry, Rx, T);
    mat3_mul(Rz, T, R);
    if (dR) {
        double dRx[9] = {0, 0, 0, 0, -sr, -cr, 0, cr, -sr};
        double dRy[9] = {-sp, 0, cp, 0, 0, 0, -cp, 0, -sp};
        double dRz[9] = {-sy, -cy, 0, cy, -sy, 0, 0, 0, 0};
        mat3_mul(Ry, dRx, T); mat3_mul(Rz, T, dR + 0);
        mat3_mul(dRy, Rx, T); mat3_mul(Rz, T, dR + 9);
        mat3_mul(Ry, Rx, T);  mat3_mul(dRz, T, dR + 18);
    }
}

static void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

/* skew(a) such that skew(a) b = a x b */
static void skew3(const double *a, double *S) {
    S[0] = 0;     S[1] = -a[2]; S[2] = a[1];
    S[3] = a[2];  S[4] = 0;     S[5] = -a[0];
    S[6] = -a[1]; S[7] = a[0];  S[8] = 0;
}

/* Continuous SRBD dynamics f(x,u):
 *   pdot = v;  Thetadot = E(Theta)^{-1} w  (ZYX);  vdot = (1/m) sum_j c_j f_j + g;
 *   wdot = I^{-1} ( R^T sum_j c_j (r_j - p) x f_j  -  w x I w ).                      */
void oracle_srbd_f(const oracle_srbd_params *P, const double *x, const double *u,
                   const double *feet /*[4][3]*/, const uint8_t *contact /*[4]*/, double *xd) {
    const double *pos = x, *th = x + 3, *v = x + 6, *w = x + 9;
    double R[9], Ii[9];
    rot_zyx(th, R, NULL);
    mat3_inv(P->inertia, Ii);
    double sr = sin(th[0]), cr = cos(th[0]), cp = cos(th[1]), tp = tan(th[1]);
    xd[0] = v[0]; xd[1] = v[1]; xd[2] = v[2];
    xd[3] = w[0] + sr * tp * w[1] + cr * tp * w[2];
    xd[4] = cr * w[1] - sr * w[2];
    xd[5] = (sr * w[1] + cr * w[2]) / cp;
    double F[3] = {0, 0, 0}, tau_w[3] = {0, 0, 0};
    for (int j = 0; j < NFEET; ++j) {
        if (!contact[j]) continue;
        const double *f = u + 3 * j;
        double rr[3] = {feet[3 * j] - pos[0], feet[3 * j + 1] - pos[1], feet[3 * j + 2] - pos[2]};
        double t[3];
        cross3(rr, f, t);
        for (int a = 0; a < 3; ++a) { F[a] += f[a]; tau_w[a] += t[a]; }
    }
    for (int a = 0; a < 3; ++a) xd[6 + a] = F[a] / P->mass + P->gravity[a];
    double tau_b[3], Iw[3], wxIw[3], rhs[3];
    for (int a = 0; a < 3; ++a) {
        tau_b[a] = R[0 + a] * tau_w[0] + R[3 + a] * tau_w[1] + R[6 + a] * tau_w[2]; /* R^T tau */
        Iw[a] = P->inertia[3 * a] * w[0] + P->inertia[3 * a + 1] * w[1] + P->inertia[3 * a + 2] * w[2];
    }
    cross3(w, Iw, wxIw);
    for (int a = 0; a < 3; ++a) rhs[a] = tau_b[a] - wxIw[a];
    for (int a = 0; a < 3; ++a) xd[9 + a] = Ii[3 * a] * rhs[0] + Ii[3 * a + 1] * rhs[1] + Ii[3 * a + 2] * rhs[2];
}

/* Analytic Jacobians Fx = df/dx (12x12), Fu = df/du (12x12) of the continuous dynamics. */
void oracle_srbd_jac(const oracle_srbd_params *P, const double *x, const double *u,
                     const double *feet, const uint8_t *contact, double *Fx, double *Fu) {
    const double *pos = x, *th = x + 3, *w = x + 9;
    memset(Fx, 0, sizeof(double) * NX * NX);
    memset(Fu, 0, sizeof(double) * NX * NU);
    double R[9], dR[27], Ii[9];
    rot_zyx(th, R, dR);
    mat3_inv(P->inertia, Ii);
    double sr = sin(th[0]), cr = cos(th[0]), sp = sin(th[1]), cp = cos(th[1]), tp = tan(th[1]);
    /* pdot = v */
    for (int a = 0; a < 3; ++a) Fx[IDX2(a, 6 + a, NX)] = 1.0;
    /* Thetadot = E^{-1}(roll,pitch) w */
    Fx[IDX2(3, 3, NX)] = cr * tp * w[1] - sr * tp * w[2];
    Fx[IDX2(3, 4, NX)] = (sr * w[1] + cr * w[2]) / (cp * cp);
    Fx[IDX2(4, 3, NX)] = -sr * w[1] - cr * w[2];
    Fx[IDX2(5, 3, NX)] = (cr * w[1] - sr * w[2]) / cp;
    Fx[IDX2(5, 4, NX)] = (sr * w[1] + cr * w[2]) * sp / (cp * cp);
    Fx[IDX2(3, 9, NX)] = 1.0; Fx[IDX2(3, 10, NX)] = sr * tp; Fx[IDX2(3, 11, NX)] = cr * tp;
    Fx[IDX2(4, 10, NX)] = cr;  Fx[IDX2(4, 11, NX)] = -sr;
    Fx[IDX2(5, 10, NX)] = sr / cp; Fx[IDX2(5, 11, NX)] = cr / cp;
    /* vdot = sum c_j f_j / m + g */
    for (int j = 0; j < NFEET; ++j)
        if (contact[j])
            for (int a = 0; a < 3; ++a) Fu[IDX2(6 + a, 3 * j + a, NU)] = 1.0 / P->mass;
    /* wdot = I^{-1}(R^T tau_w - w x I w), tau_w = sum c_j (r_j - p) x f_j */
    double tau_w[3] = {0, 0, 0}, dtau_dp[9] = {0};
    for (int j = 0; j < NFEET; ++j) {
        if (!contact[j]) continue;
        const double *f = u + 3 * j;
        double rr[3] = {feet[3 * j] - pos[0], feet[3 * j + 1] - pos[1], feet[3 * j + 2] - pos[2]};
        double t[3], Sf[9], Sr[9];
        cross3(rr, f, t);
        for (int a = 0; a < 3; ++a) tau_w[a] += t[a];
        skew3(f, Sf);                /* d[(r - p) x f]/dp = skew(f) */
        for (int a = 0; a < 9; ++a) dtau_dp[a] += Sf[a];
        skew3(rr, Sr);               /* d[(r - p) x f]/df = skew(r - p) */
        double RtS[9], IiRtS[9], Rt[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) Rt[3 * a + b] = R[3 * b + a];
        mat3_mul(Rt, Sr, RtS);
        mat3_mul(Ii, RtS, IiRtS);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) Fu[IDX2(9 + a, 3 * j + b, NU)] = IiRtS[3 * a + b];
    }
    double Rt[9], M1[9], M2[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Rt[3 * a + b] = R[3 * b + a];
    mat3_mul(Rt, dtau_dp, M1);
    mat3_mul(Ii, M1, M2);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Fx[IDX2(9 + a, b, NX)] = M2[3 * a + b];
    for (int k = 0; k < 3; ++k) { /* d(R^T tau_w)/dTheta_k = (dR/dTheta_k)^T tau_w */
        double col[3];
        for (int a = 0; a < 3; ++a)
            col[a] = dR[9 * k + 0 + a] * tau_w[0] + dR[9 * k + 3 + a] * tau_w[1] + dR[9 * k + 6 + a] * tau_w[2];
        for (int a = 0; a < 3; ++a)
            Fx[IDX2(9 + a, 3 + k, NX)] = Ii[3 * a] * col[0] + Ii[3 * a + 1] * col[1] + Ii[3 * a + 2] * col[2];
    }
    /* d(-w x I w)/dw = -(skew(w) I - skew(I w)) */
    double Iw[3], Sw[9], SIw[9], SwI[9], D[9];
    for (int a = 0; a < 3; ++a)
        Iw[a] = P->inertia[3 * a] * w[0] + P->inertia[3 * a + 1] * w[1] + P->inertia[3 * a + 2] * w[2];
    skew3(w, Sw);
    skew3(Iw, SIw);
    mat3_mul(Sw, P->inertia, SwI);
    for (int a = 0; a < 9; ++a) D[a] = -(SwI[a] - SIw[a]);
    double IiD[9];
    mat3_mul(Ii, D, IiD);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Fx[IDX2(9 + a, 9 + b, NX)] = IiD[3 * a + b];
}

/* Explicit Euler step h(x,u) = x + dt f(x,u) (reading R14). */
void oracle_srbd_h(const oracle_srbd_params *P, const double *x, const double *u,
                   const double *feet, const uint8_t *contact, double *xn) {
    double xd[NX];
    oracle_srbd_f(P, x, u, feet, contact, xd);
    for (int a = 0; a < NX; ++a) xn[a] = x[a] + P->dt * xd[a];
}

/* ------------------------------------------------------------------------- */
/* relaxed barrier (sign reading R11: feasible <=> xi > 0)        */
/* ------------------------------------------------------------------------- */
double oracle_barrier(double xi, double mu, double delta) {
    if (xi >= delta) return -mu * log(xi);
    double t = (xi - 2.0 * delta) / delta;
    return 0.5 * mu * (t * t - 1.0) - mu * log(delta);
}
double oracle_barrier_d1(double xi, double mu, double delta) {
    if (xi >= delta) return -mu / xi;
    return mu * (xi - 2.0 * delta) / (delta * delta);
}
double oracle_barrier_d2(double xi, double mu, double delta) {
    if (xi >= delta) return mu / (xi * xi);
    return mu / (delta * delta);
}

/* The six linear constraints xi_c(f) = g_c . f_j + h_c per stance foot j: friction
 * pyramid (4) and normal-force bounds (2).  Gradient written into g[3], offset h. */
static void foot_constraint(const oracle_srbd_params *P, int c, double *g, double *h) {
    double mu = P->mu_friction;
    g[0] = g[1] = g[2] = 0; *h = 0;
    switch (c) {
    case 0: g[0] = -1; g[2] = mu; break;         /* mu fz - fx */
    case 1: g[0] = 1;  g[2] = mu; break;         /* mu fz + fx */
    case 2: g[1] = -1; g[2] = mu; break;         /* mu fz - fy */
    case 3: g[1] = 1;  g[2] = mu; break;         /* mu fz + fy */
    case 4: g[2] = 1;  *h = -P->f_min; break;    /* fz - fmin  */
    default: g[2] = -1; *h = P->f_max; break;    /* fmax - fz  */
    }
}

static double u_weight(const oracle_srbd_params *P, const uint8_t *contact, int a) {
    return contact[a / 3] ? P->w_u_stance : P->w_u_swing;
}

/* Stage cost l_i (P:290-297 NLS form + barriers on stance feet), i = 0..N. */
static double stage_cost(const oracle_srbd_params *P, const double *x, const double *u,
                         const double *xr, const double *ur, const uint8_t *contact) {
    double J = 0;
    for (int a = 0; a < NX; ++a) J += 0.5 * P->w_x[a] * (x[a] - xr[a]) * (x[a] - xr[a]);
    for (int a = 0; a < NU; ++a) {
        double d = u[a] - (ur ? ur[a] : 0.0);
        J += 0.5 * u_weight(P, contact, a) * d * d;
    }
    for (int j = 0; j < NFEET; ++j) {
        if (!contact[j]) continue;
        for (int cc = 0; cc < 6; ++cc) {
            double g[3], h;
            foot_constraint(P, cc, g, &h);
            double xi = g[0] * u[3 * j] + g[1] * u[3 * j + 1] + g[2] * u[3 * j + 2] + h;
            J += oracle_barrier(xi, P->barrier_mu, P->barrier_delta);
        }
    }
    return J;
}

static double term_cost(const oracle_srbd_params *P, const double *x, const double *xr) {
    double J = 0;
    for (int a = 0; a < NX; ++a) J += 0.5 * P->w_x_term[a] * (x[a] - xr[a]) * (x[a] - xr[a]);
    return J;
}

static int pitch_ok(const double *x) { return fabs(x[4]) < PITCH_GUARD && isfinite(x[4]); }

/* Linearise + quadraticise at the iterate (x,u,lam):
 *   A = I + dt Fx, B = dt Fu, b_i = h(x_i,u_i) - x_{i+1};
 *   Q = W_x, S = 0, R = W_u + sum_c B''(xi_c) grad xi_c grad xi_c^T (GN);
 *   q_i = W_x (x_i - xref_i) + A_i^T lam_{i+1} - lam_i                 (q = grad_x L)
 *   r_i = W_u (u_i - uref_i) + sum_c B'(xi_c) grad xi_c + B_i^T lam_{i+1}  (r = grad_u L)
 *   P_{N+1} = W_N, p_{N+1} = W_N (x_{N+1} - xref_{N+1}) - lam_{N+1},  dx0 = xhat0 - x_0.
 * Returns 0, or -1 if the iterate is outside the Euler-angle guard or not finite. */
int oracle_srbd_linearize(const oracle_srbd_params *P, int N,
                          const double *x, const double *u, const double *lam,
                          const double *x0, const double *xref, const double *uref,
                          const uint8_t *contact, const double *feet,
                          double *A, double *Bm, double *c, double *Q, double *R, double *S,
                          double *q, double *r, double *Pt, double *pt, double *dx0) {
    for (int i = 0; i <= N + 1; ++i)
        for (int a = 0; a < NX; ++a)
            if (!isfinite(x[i * NX + a]) || !isfinite(lam[i * NX + a])) return -1;
    for (int i = 0; i <= N; ++i) {
        if (!pitch_ok(x + i * NX)) return -1;
        for (int a = 0; a < NU; ++a)
            if (!isfinite(u[i * NU + a])) return -1;
    }
    double Fx[NX * NX], Fu[NX * NU];
    for (int i = 0; i <= N; ++i) {
        const double *xi = x + i * NX, *ui = u + i * NU, *fi = feet + i * 12;
        const uint8_t *ci = contact + i * 4;
        const double *ln = lam + (i + 1) * NX, *li = lam + i * NX;
        double *Ai = A + (size_t)i * NX * NX, *Bi = Bm + (size_t)i * NX * NU;
        double *Qi = Q + (size_t)i * NX * NX, *Ri = R + (size_t)i * NU * NU, *Si = S + (size_t)i * NU * NX;
        oracle_srbd_jac(P, xi, ui, fi, ci, Fx, Fu);
        for (int a = 0; a < NX; ++a)
            for (int b = 0; b < NX; ++b) Ai[IDX2(a, b, NX)] = (a == b ? 1.0 : 0.0) + P->dt * Fx[IDX2(a, b, NX)];
        for (int a = 0; a < NX; ++a)
            for (int b = 0; b < NU; ++b) Bi[IDX2(a, b, NU)] = P->dt * Fu[IDX2(a, b, NU)];
        double xn[NX];
        oracle_srbd_h(P, xi, ui, fi, ci, xn);
        for (int a = 0; a < NX; ++a) c[i * NX + a] = xn[a] - x[(i + 1) * NX + a];
        memset(Qi, 0, sizeof(double) * NX * NX);
        memset(Ri, 0, sizeof(double) * NU * NU);
        memset(Si, 0, sizeof(double) * NU * NX);
        for (int a = 0; a < NX; ++a) Qi[IDX2(a, a, NX)] = P->w_x[a];
        for (int a = 0; a < NU; ++a) Ri[IDX2(a, a, NU)] = u_weight(P, ci, a);
        double rg[NU];
        for (int a = 0; a < NU; ++a) rg[a] = u_weight(P, ci, a) * (ui[a] - (uref ? uref[i * NU + a] : 0.0));
        for (int j = 0; j < NFEET; ++j) {
            if (!ci[j]) continue;
            for (int cc = 0; cc < 6; ++cc) {
                double g[3], h;
                foot_constraint(P, cc, g, &h);
                double xi_c = g[0] * ui[3 * j] + g[1] * ui[3 * j + 1] + g[2] * ui[3 * j + 2] + h;
                double d1 = oracle_barrier_d1(xi_c, P->barrier_mu, P->barrier_delta);
                double d2 = oracle_barrier_d2(xi_c, P->barrier_mu, P->barrier_delta);
                for (int a = 0; a < 3; ++a) {
                    rg[3 * j + a] += d1 * g[a];
                    for (int b = 0; b < 3; ++b) Ri[IDX2(3 * j + a, 3 * j + b, NU)] += d2 * g[a] * g[b];
                }
            }
        }
        for (int a = 0; a < NX; ++a) {
            double s = P->w_x[a] * (xi[a] - xref[i * NX + a]) - li[a];
            for (int t = 0; t < NX; ++t) s += Ai[IDX2(t, a, NX)] * ln[t];
            q[i * NX + a] = s;
        }
        for (int a = 0; a < NU; ++a) {
            double s = rg[a];
            for (int t = 0; t < NX; ++t) s += Bi[IDX2(t, a, NU)] * ln[t];
            r[i * NU + a] = s;
        }
    }
    memset(Pt, 0, sizeof(double) * NX * NX);
    for (int a = 0; a < NX; ++a) {
        Pt[IDX2(a, a, NX)] = P->w_x_term[a];
        pt[a] = P->w_x_term[a] * (x[(N + 1) * NX + a] - xref[(N + 1) * NX + a]) - lam[(N + 1) * NX + a];
        dx0[a] = x0[a] - x[a];
    }
    return 0;
}

/* Total cost J(x,u) = sum_{i=0}^{N} l_i + l_{N+1} (Eq. 1 objective), barriers included. */
double oracle_srbd_cost(const oracle_srbd_params *P, int N, const double *x, const double *u,
                        const double *xref, const double *uref, const uint8_t *contact) {
    double J = 0;
    for (int i = 0; i <= N; ++i)
        J += stage_cost(P, x + i * NX, u + i * NU, xref + i * NX, uref ? uref + i * NU : NULL, contact + i * 4);
    return J + term_cost(P, x + (N + 1) * NX, xref + (N + 1) * NX);
}

/* theta = sum_{i=0}^{N} ||x_{i+1} - h(x_i,u_i)||_2 + ||xhat0 - x_0||_2 (Eq. 17, reading R9). */
double oracle_srbd_theta(const oracle_srbd_params *P, int N, const double *x, const double *u,
                         const double *x0, const uint8_t *contact, const double *feet) {
    double th = 0, d0 = 0;
    for (int a = 0; a < NX; ++a) d0 += (x0[a] - x[a]) * (x0[a] - x[a]);
    th += sqrt(d0);
    for (int i = 0; i <= N; ++i) {
        double xn[NX], s = 0;
        oracle_srbd_h(P, x + i * NX, u + i * NU, feet + i * 12, contact + i * 4, xn);
        for (int a = 0; a < NX; ++a) {
            double d = x[(i + 1) * NX + a] - xn[a];
            s += d * d;
        }
        th += sqrt(s);
    }
    return th;
}

/* Directional derivative of the cost, grad J(x,u) . (dx,du) (descent test, reading R10). */
double oracle_srbd_cost_slope(const oracle_srbd_params *P, int N, const double *x, const double *u,
                              const double *xref, const double *uref, const uint8_t *contact,
                              const double *dx, const double *du) {
    double g = 0;
    for (int i = 0; i <= N; ++i) {
        const double *xi = x + i * NX, *ui = u + i * NU;
        const uint8_t *ci = contact + i * 4;
        for (int a = 0; a < NX; ++a) g += P->w_x[a] * (xi[a] - xref[i * NX + a]) * dx[i * NX + a];
        for (int a = 0; a < NU; ++a)
            g += u_weight(P, ci, a) * (ui[a] - (uref ? uref[i * NU + a] : 0.0)) * du[i * NU + a];
        for (int j = 0; j < NFEET; ++j) {
            if (!ci[j]) continue;
            for (int cc = 0; cc < 6; ++cc) {
                double gg[3], h;
                foot_constraint(P, cc, gg, &h);
                double xi_c = gg[0] * ui[3 * j] + gg[1] * ui[3 * j + 1] + gg[2] * ui[3 * j + 2] + h;
                double d1 = oracle_barrier_d1(xi_c, P->barrier_mu, P->barrier_delta);
                g += d1 * (gg[0] * du[i * NU + 3 * j] + gg[1] * du[i * NU + 3 * j + 1] + gg[2] * du[i * NU + 3 * j + 2]);
            }
        }
    }
    for (int a = 0; a < NX; ++a)
        g += P->w_x_term[a] * (x[(N + 1) * NX + a] - xref[(N + 1) * NX + a]) * dx[(N + 1) * NX + a];
    return g;
}

/* Filter acceptance (constants reading R10).  Returns 1 if accepted.
 *  theta0 > theta_max : "reject the step if it further increases theta"  -> accept iff tha <= th0
 *  else, descent (g<0): Armijo  J(a) <= J0 + c1 a g
 *  else               : "at least the cost or theta is decreased"  -> J(a) < J0 or tha < th0 */
static int filter_accept(double J0, double th0, double g, double Ja, double tha,
                         double alpha, double c1, double theta_max) {
    if (!(isfinite(Ja) && isfinite(tha))) return 0;
    if (th0 > theta_max) return tha <= th0;
    if (g < 0) return Ja <= J0 + c1 * alpha * g;
    return (Ja < J0) || (tha < th0);
}

/* Parallel-grid filter line search and the linear update (Eq. 16).
 * Writes per-alpha J and theta into Jal/thal if non-NULL (n_alpha entries) and the
 * baseline (J0, theta0, slope) into base[3] if non-NULL.  Returns the index j of the
 * accepted alpha = 2^-j, or -1 if every trial was rejected (alpha = 0, no step). */
int oracle_srbd_line_search(const oracle_srbd_params *P, int N, int n_alpha, double c1, double theta_max,
                            const double *x, const double *u, const double *x0,
                            const double *xref, const double *uref,
                            const uint8_t *contact, const double *feet,
                            const double *dx, const double *du,
                            double *Jal, double *thal, double *base) {
    double J0 = oracle_srbd_cost(P, N, x, u, xref, uref, contact);
    double th0 = oracle_srbd_theta(P, N, x, u, x0, contact, feet);
    double g = oracle_srbd_cost_slope(P, N, x, u, xref, uref, contact, dx, du);
    if (base) { base[0] = J0; base[1] = th0; base[2] = g; }
    double *xa = malloc(sizeof(double) * (N + 2) * NX), *ua = malloc(sizeof(double) * (N + 1) * NU);
    int best = -1;
    for (int j = 0; j < n_alpha; ++j) {
        double alpha = ldexp(1.0, -j);
        int ok = 1;
        for (int t = 0; t < (N + 2) * NX; ++t) xa[t] = x[t] + alpha * dx[t];
        for (int t = 0; t < (N + 1) * NU; ++t) ua[t] = u[t] + alpha * du[t];
        for (int i = 0; i <= N; ++i) ok &= pitch_ok(xa + i * NX);
        double Ja = ok ? oracle_srbd_cost(P, N, xa, ua, xref, uref, contact) : INFINITY;
        double tha = ok ? oracle_srbd_theta(P, N, xa, ua, x0, contact, feet) : INFINITY;
        if (Jal) Jal[j] = Ja;
        if (thal) thal[j] = tha;
        if (best < 0 && filter_accept(J0, th0, g, Ja, tha, alpha, c1, theta_max)) best = j;
    }
    free(xa); free(ua);
    return best;
}

/* One SQP/RTI iteration (one iteration per control tick): linearise -> LQ solve
 * (Riccati) -> dual update -> filter line search -> update x,u,lam in place (Eq. 16).
 * stats[5] = {cost, theta, alpha, accepted, info}.  dirs (dx,du,dlam) optional out. */
/* The same iteration with a Levenberg-Marquardt shift rho added to every R_i after the
 * linearisation (the ladder of pdilqr_solve, SPEC S:75 / S:362, reading R28). */
int oracle_srbd_step_rho(const oracle_srbd_params *P, int N, int n_alpha, double c1, double theta_max, double rho,
                         double *x, double *u, double *lam, const double *x0,
                         const double *xref, const double *uref,
                         const uint8_t *contact, const double *feet,
                         double *stats, double *dx_out, double *du_out, double *dlam_out);

int oracle_srbd_step(const oracle_srbd_params *P, int N, int n_alpha, double c1, double theta_max,
                     double *x, double *u, double *lam, const double *x0,
                     const double *xref, const double *uref,
                     const uint8_t *contact, const double *feet,
                     double *stats, double *dx_out, double *du_out, double *dlam_out) {
    return oracle_srbd_step_rho(P, N, n_alpha, c1, theta_max, 0.0, x, u, lam, x0, xref, uref, contact, feet,
                                stats, dx_out, du_out, dlam_out);
}

int oracle_srbd_step_rho(const oracle_srbd_params *P, int N, int n_alpha, double c1, double theta_max, double rho,
                         double *x, double *u, double *lam, const double *x0,
                         const double *xref, const double *uref,
                         const uint8_t *contact, const double *feet,
                         double *stats, double *dx_out, double *du_out, double *dlam_out) {
    const int n = NX, m = NU;
    const size_t S1 = (size_t)(N + 1);
    double *A = malloc(sizeof(double) * S1 * n * n), *Bm = malloc(sizeof(double) * S1 * n * m);
    double *c = malloc(sizeof(double) * S1 * n), *Q = malloc(sizeof(double) * S1 * n * n);
    double *R = malloc(sizeof(double) * S1 * m * m), *S = malloc(sizeof(double) * S1 * m * n);
    double *q = malloc(sizeof(double) * S1 * n), *r = malloc(sizeof(double) * S1 * m);
    double Pt[NX * NX], pt[NX], d0[NX];
    double *dx = malloc(sizeof(double) * (S1 + 1) * n), *du = malloc(sizeof(double) * S1 * m);
    double *dl = malloc(sizeof(double) * (S1 + 1) * n);
    double theta_thr = theta_max > 0 ? theta_max : 1e-2 * (N + 1);
    int info = oracle_srbd_linearize(P, N, x, u, lam, x0, xref, uref, contact, feet,
                                     A, Bm, c, Q, R, S, q, r, Pt, pt, d0);
    if (info == 0 && rho != 0.0)
        for (size_t i = 0; i < S1; ++i)
            for (int a = 0; a < m; ++a) R[i * m * m + IDX2(a, a, m)] += rho;
    if (info == 0) info = oracle_solve_lq(N, n, m, A, Bm, c, Q, R, S, q, r, Pt, pt, d0, dx, du, dl,
                                          NULL, NULL, NULL, NULL);
    if (info == 0) {
        for (size_t t = 0; t < (S1 + 1) * n; ++t)
            if (!isfinite(dx[t]) || !isfinite(dl[t])) info = -1;
        for (size_t t = 0; t < S1 * m; ++t)
            if (!isfinite(du[t])) info = -1;
    }
    double J0 = oracle_srbd_cost(P, N, x, u, xref, uref, contact);
    double th0 = oracle_srbd_theta(P, N, x, u, x0, contact, feet);
    double alpha = 0, Jn = J0, thn = th0;
    int accepted = 0;
    if (info == 0) {
        double Jal[32], thal[32];
        int na = n_alpha > 32 ? 32 : n_alpha;
        int j = oracle_srbd_line_search(P, N, na, c1, theta_thr, x, u, x0, xref, uref, contact, feet,
                                        dx, du, Jal, thal, NULL);
        if (j >= 0) {
            alpha = ldexp(1.0, -j);
            accepted = 1;
            Jn = Jal[j];
            thn = thal[j];
            for (size_t t = 0; t < (S1 + 1) * n; ++t) { x[t] += alpha * dx[t]; lam[t] += alpha * dl[t]; }
            for (size_t t = 0; t < S1 * m; ++t) u[t] += alpha * du[t];
        }
    }
    if (stats) { stats[0] = Jn; stats[1] = thn; stats[2] = alpha; stats[3] = accepted; stats[4] = info; }
    if (dx_out) memcpy(dx_out, dx, sizeof(double) * (S1 + 1) * n);
    if (du_out) memcpy(du_out, du, sizeof(double) * S1 * m);
    if (dlam_out) memcpy(dlam_out, dl, sizeof(double) * (S1 + 1) * n);
    free(A); free(Bm); free(c); free(Q); free(R); free(S); free(q); free(r);
    free(dx); free(du); free(dl);
    return info;
}

/* Batched SRBD step over B instances (batch-outermost arrays), OpenMP over instances. */
void oracle_srbd_step_batch(const oracle_srbd_params *P, int Bn, int N, int n_alpha, double c1,
                            double theta_max, double *x, double *u, double *lam, const double *x0,
                            const double *xref, const double *uref, const uint8_t *contact,
                            const double *feet, double *stats, int nthreads) {
    const size_t S1 = (size_t)(N + 1);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int b = 0; b < Bn; ++b)
        oracle_srbd_step(P, N, n_alpha, c1, theta_max, x + b * (S1 + 1) * NX, u + b * S1 * NU,
                         lam + b * (S1 + 1) * NX, x0 + (size_t)b * NX, xref + b * (S1 + 1) * NX,
                         uref ? uref + b * S1 * NU : NULL, contact + b * S1 * 4, feet + b * S1 * 12,
                         stats + (size_t)b * 5, NULL, NULL, NULL);
}

/* Batched linearisation (used by parity tests of pdilqr_linearize). */
void oracle_srbd_linearize_batch(const oracle_srbd_params *P, int Bn, int N,
                                 const double *x, const double *u, const double *lam,
                                 const double *x0, const double *xref, const double *uref,
                                 const uint8_t *contact, const double *feet,
                                 double *A, double *Bm, double *c, double *Q, double *R, double *S,
                                 double *q, double *r, double *Pt, double *pt, double *dx0,
                                 int32_t *info, int nthreads) {
    const size_t S1 = (size_t)(N + 1);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int b = 0; b < Bn; ++b)
        info[b] = oracle_srbd_linearize(
            P, N, x + b * (S1 + 1) * NX, u + b * S1 * NU, lam + b * (S1 + 1) * NX, x0 + (size_t)b * NX,
            xref + b * (S1 + 1) * NX, uref ? uref + b * S1 * NU : NULL, contact + b * S1 * 4,
            feet + b * S1 * 12, A + b * S1 * NX * NX, Bm + b * S1 * NX * NU, c + b * S1 * NX,
            Q + b * S1 * NX * NX, R + b * S1 * NU * NU, S + b * S1 * NU * NX, q + b * S1 * NX,
            r + b * S1 * NU, Pt + (size_t)b * NX * NX, pt + (size_t)b * NX, dx0 + (size_t)b * NX);
}

/* ------------------------------------------------------------------------- */
/* Centralized multi-robot SRBD model (NEXT-3) */
/* ------------------------------------------------------------------------- */
/* R robots share one OCP: state x = [x_robot0 (12) .. x_robot{R-1}], input likewise, contact
 * [4R], footholds [4R][3].  Dynamics and the per-robot cost are R copies of the SRBD model above
 * (block-diagonal A, B, Q, R; S = 0).  Coupling: a collision-avoidance penalty ("a quadratic
 * penalty term"; "smooth quadratic penalty (softplus smoothing)") on every robot pair
 * (a < b) at every node i = 0..N+1:
 *   d = sqrt(|p_a - p_b|_xy^2 + eta^2)  (planar CoM distance, eta = 1e-3 regularises d = 0),
 *   eps = softplus_k(d_min - d) = log(1 + exp(k (d_min - d))) / k,   cost 1/2 w eps^2;
 * Gauss-Newton: Hessian w grad eps grad eps^T, gradient w eps grad eps, with
 *   grad_{p_a} eps = -sigma(k (d_min - d)) (p_a - p_b) / d,  grad_{p_b} eps = -grad_{p_a} eps. */
typedef struct {
    int n_robots;
    double d_min, weight, sharpness;
} oracle_multi_params;

#define COLL_ETA 1e-3

/* One pair term at positions pa, pb (xy): eps and grad eps w.r.t. (pa_x, pa_y, pb_x, pb_y). */
static double coll_pair(const oracle_multi_params *M, const double *pa, const double *pb, double *g4) {
    double dx = pa[0] - pb[0], dy = pa[1] - pb[1];
    double d = sqrt(dx * dx + dy * dy + COLL_ETA * COLL_ETA);
    double s = M->sharpness * (M->d_min - d);
    double eps = (s > 0 ? s + log1p(exp(-s)) : log1p(exp(s))) / M->sharpness;
    double sig = 1.0 / (1.0 + exp(-s));
    g4[0] = -sig * dx / d; g4[1] = -sig * dy / d;
    g4[2] = sig * dx / d;  g4[3] = sig * dy / d;
    return eps;
}

/* Collision cost of one node (sum over pairs of 1/2 w eps^2). */
double oracle_multi_coll_cost(const oracle_multi_params *M, const double *x /* [12 R] */) {
    double J = 0, g4[4];
    for (int a = 0; a < M->n_robots; ++a)
        for (int b = a + 1; b < M->n_robots; ++b) {
            double e = coll_pair(M, x + 12 * a, x + 12 * b, g4);
            J += 0.5 * M->weight * e * e;
        }
    return J;
}

/* Add the Gauss-Newton collision terms of one node to H (n x n, ld n) and h (n). */
static void coll_gn(const oracle_multi_params *M, const double *x, double *H, double *h) {
    const int n = 12 * M->n_robots;
    for (int a = 0; a < M->n_robots; ++a)
        for (int b = a + 1; b < M->n_robots; ++b) {
            double g4[4];
            double e = coll_pair(M, x + 12 * a, x + 12 * b, g4);
            int idx[4] = {12 * a, 12 * a + 1, 12 * b, 12 * b + 1};
            for (int s = 0; s < 4; ++s) {
                h[idx[s]] += M->weight * e * g4[s];
                for (int t = 0; t < 4; ++t) H[IDX2(idx[s], idx[t], n)] += M->weight * g4[s] * g4[t];
            }
        }
}

/* Linearise + quadraticise the centralized OCP at (x, u, lam): per robot the SRBD linearisation
 * of oracle_srbd_linearize on that robot's slices (block-diagonal placement; q, r with the
 * multiplier terms of the robot's own constraints), plus the collision terms at nodes
 * 0..N (into Q_i, q_i) and N+1 (into P_{N+1}, p_{N+1}).  Returns 0 or -1 (any robot invalid). */
int oracle_multi_linearize(const oracle_srbd_params *P, const oracle_multi_params *M, int N,
                           const double *x, const double *u, const double *lam,
                           const double *x0, const double *xref, const double *uref,
                           const uint8_t *contact, const double *feet,
                           double *A, double *Bm, double *c, double *Q, double *R, double *S,
                           double *q, double *r, double *Pt, double *pt, double *dx0) {
    const int Rn = M->n_robots, n = 12 * Rn;
    const size_t S1 = (size_t)(N + 1), S2 = S1 + 1, nn = (size_t)n * n;
    memset(A, 0, sizeof(double) * S1 * nn); memset(Bm, 0, sizeof(double) * S1 * nn);
    memset(Q, 0, sizeof(double) * S1 * nn); memset(R, 0, sizeof(double) * S1 * nn);
    memset(S, 0, sizeof(double) * S1 * nn); memset(Pt, 0, sizeof(double) * nn);
    /* per-robot slices and outputs */
    double *xs = malloc(sizeof(double) * S2 * 12), *us = malloc(sizeof(double) * S1 * 12);
    double *ls = malloc(sizeof(double) * S2 * 12), *xrs = malloc(sizeof(double) * S2 * 12);
    double *urs = malloc(sizeof(double) * S1 * 12), *fs = malloc(sizeof(double) * S1 * 12);
    uint8_t *cs = malloc(S1 * 4);
    double *a1 = malloc(sizeof(double) * S1 * 144), *b1 = malloc(sizeof(double) * S1 * 144);
    double *c1 = malloc(sizeof(double) * S1 * 12), *q1m = malloc(sizeof(double) * S1 * 144);
    double *r1m = malloc(sizeof(double) * S1 * 144), *s1m = malloc(sizeof(double) * S1 * 144);
    double *q1 = malloc(sizeof(double) * S1 * 12), *r1 = malloc(sizeof(double) * S1 * 12);
    double pt1m[144], pt1[12], d01[12];
    int info = 0;
    for (int k = 0; k < Rn && info == 0; ++k) {
        for (size_t i = 0; i < S2; ++i)
            for (int a = 0; a < 12; ++a) {
                xs[i * 12 + a] = x[i * n + 12 * k + a];
                ls[i * 12 + a] = lam[i * n + 12 * k + a];
                xrs[i * 12 + a] = xref[i * n + 12 * k + a];
            }
        for (size_t i = 0; i < S1; ++i) {
            for (int a = 0; a < 12; ++a) {
                us[i * 12 + a] = u[i * n + 12 * k + a];
                urs[i * 12 + a] = uref ? uref[i * n + 12 * k + a] : 0.0;
                fs[i * 12 + a] = feet[i * 12 * Rn + 12 * k + a];
            }
            for (int j = 0; j < 4; ++j) cs[i * 4 + j] = contact[i * 4 * Rn + 4 * k + j];
        }
        double x0s[12];
        for (int a = 0; a < 12; ++a) x0s[a] = x0[12 * k + a];
        info = oracle_srbd_linearize(P, N, xs, us, ls, x0s, xrs, urs, cs, fs,
                                     a1, b1, c1, q1m, r1m, s1m, q1, r1, pt1m, pt1, d01);
        if (info) break;
        for (size_t i = 0; i < S1; ++i) {
            for (int a = 0; a < 12; ++a) {
                for (int bb = 0; bb < 12; ++bb) {
                    size_t o = i * nn + IDX2(12 * k + a, 12 * k + bb, n);
                    A[o] = a1[i * 144 + IDX2(a, bb, 12)];
                    Bm[o] = b1[i * 144 + IDX2(a, bb, 12)];
                    Q[o] = q1m[i * 144 + IDX2(a, bb, 12)];
                    R[o] = r1m[i * 144 + IDX2(a, bb, 12)];
                }
                c[i * n + 12 * k + a] = c1[i * 12 + a];
                q[i * n + 12 * k + a] = q1[i * 12 + a];
                r[i * n + 12 * k + a] = r1[i * 12 + a];
            }
        }
        for (int a = 0; a < 12; ++a) {
            for (int bb = 0; bb < 12; ++bb) Pt[IDX2(12 * k + a, 12 * k + bb, n)] = pt1m[IDX2(a, bb, 12)];
            pt[12 * k + a] = pt1[a];
            dx0[12 * k + a] = d01[a];
        }
    }
    if (info == 0) {
        for (size_t i = 0; i < S1; ++i) coll_gn(M, x + i * n, Q + i * nn, q + i * n);
        coll_gn(M, x + S1 * n, Pt, pt);
    }
    free(xs); free(us); free(ls); free(xrs); free(urs); free(fs); free(cs);
    free(a1); free(b1); free(c1); free(q1m); free(r1m); free(s1m); free(q1); free(r1);
    return info;
}

/* Copy robot k's slices (x, u of stride 12 R) of a trajectory into single-robot arrays. */
static void robot_slice(int Rn, int k, int N, const double *x, const double *u, const uint8_t *contact,
                        const double *feet, const double *xref, const double *uref,
                        double *xs, double *us, uint8_t *cs, double *fs, double *xrs, double *urs) {
    const int n = 12 * Rn;
    for (int i = 0; i <= N + 1; ++i)
        for (int a = 0; a < 12; ++a) {
            if (xs) xs[i * 12 + a] = x[i * n + 12 * k + a];
            if (xrs) xrs[i * 12 + a] = xref[i * n + 12 * k + a];
        }
    for (int i = 0; i <= N; ++i) {
        for (int a = 0; a < 12; ++a) {
            if (us) us[i * 12 + a] = u[i * n + 12 * k + a];
            if (urs) urs[i * 12 + a] = uref ? uref[i * n + 12 * k + a] : 0.0;
            if (fs) fs[i * 12 + a] = feet[i * 12 * Rn + 12 * k + a];
        }
        if (cs) for (int j = 0; j < 4; ++j) cs[i * 4 + j] = contact[i * 4 * Rn + 4 * k + j];
    }
}

/* J = sum_k J_srbd(robot k) + sum_{i=0}^{N+1} sum_{a<b} 1/2 w eps_ab(x_i)^2. */
double oracle_multi_cost(const oracle_srbd_params *P, const oracle_multi_params *M, int N, const double *x,
                         const double *u, const double *xref, const double *uref, const uint8_t *contact) {
    const int Rn = M->n_robots, n = 12 * Rn;
    double *xs = malloc(sizeof(double) * (N + 2) * 12), *us = malloc(sizeof(double) * (N + 1) * 12);
    double *xrs = malloc(sizeof(double) * (N + 2) * 12), *urs = malloc(sizeof(double) * (N + 1) * 12);
    uint8_t *cs = malloc((size_t)(N + 1) * 4);
    double J = 0;
    for (int k = 0; k < Rn; ++k) {
        robot_slice(Rn, k, N, x, u, contact, NULL, xref, uref, xs, us, cs, NULL, xrs, urs);
        J += oracle_srbd_cost(P, N, xs, us, xrs, urs, cs);
    }
    for (int i = 0; i <= N + 1; ++i) J += oracle_multi_coll_cost(M, x + (size_t)i * n);
    free(xs); free(us); free(xrs); free(urs); free(cs);
    return J;
}

/* theta = sum_{i=0}^{N} |x_{i+1} - h(x_i, u_i)|_2 + |xhat0 - x_0|_2 over the stacked state
 * (Eq. 17, reading R9; h is the per-robot Euler step). */
double oracle_multi_theta(const oracle_srbd_params *P, const oracle_multi_params *M, int N, const double *x,
                          const double *u, const double *x0, const uint8_t *contact, const double *feet) {
    const int Rn = M->n_robots, n = 12 * Rn;
    double th = 0, d0 = 0;
    for (int a = 0; a < n; ++a) d0 += (x0[a] - x[a]) * (x0[a] - x[a]);
    th += sqrt(d0);
    for (int i = 0; i <= N; ++i) {
        double s = 0;
        for (int k = 0; k < Rn; ++k) {
            double xn[12];
            uint8_t ck[4];
            for (int j = 0; j < 4; ++j) ck[j] = contact[(size_t)i * 4 * Rn + 4 * k + j];
            oracle_srbd_h(P, x + (size_t)i * n + 12 * k, u + (size_t)i * n + 12 * k, feet + (size_t)i * 12 * Rn + 12 * k, ck, xn);
            for (int a = 0; a < 12; ++a) {
                double d = x[(size_t)(i + 1) * n + 12 * k + a] - xn[a];
                s += d * d;
            }
        }
        th += sqrt(s);
    }
    return th;
}

/* grad J . (dx, du) (descent test, reading R10): per-robot SRBD slopes + collision gradients. */
double oracle_multi_cost_slope(const oracle_srbd_params *P, const oracle_multi_params *M, int N, const double *x,
                               const double *u, const double *xref, const double *uref, const uint8_t *contact,
                               const double *dx, const double *du) {
    const int Rn = M->n_robots, n = 12 * Rn;
    double *xs = malloc(sizeof(double) * (N + 2) * 12), *us = malloc(sizeof(double) * (N + 1) * 12);
    double *xrs = malloc(sizeof(double) * (N + 2) * 12), *urs = malloc(sizeof(double) * (N + 1) * 12);
    double *dxs = malloc(sizeof(double) * (N + 2) * 12), *dus = malloc(sizeof(double) * (N + 1) * 12);
    uint8_t *cs = malloc((size_t)(N + 1) * 4);
    double g = 0;
    for (int k = 0; k < Rn; ++k) {
        robot_slice(Rn, k, N, x, u, contact, NULL, xref, uref, xs, us, cs, NULL, xrs, urs);
        robot_slice(Rn, k, N, dx, du, contact, NULL, xref, NULL, dxs, dus, NULL, NULL, NULL, NULL);
        g += oracle_srbd_cost_slope(P, N, xs, us, xrs, urs, cs, dxs, dus);
    }
    for (int i = 0; i <= N + 1; ++i) {
        const double *xi = x + (size_t)i * n, *di = dx + (size_t)i * n;
        for (int a = 0; a < Rn; ++a)
            for (int b = a + 1; b < Rn; ++b) {
                double g4[4];
                double e = coll_pair(M, xi + 12 * a, xi + 12 * b, g4);
                g += M->weight * e * (g4[0] * di[12 * a] + g4[1] * di[12 * a + 1] + g4[2] * di[12 * b] + g4[3] * di[12 * b + 1]);
            }
    }
    free(xs); free(us); free(xrs); free(urs); free(dxs); free(dus); free(cs);
    return g;
}

/* One SQP iteration of the centralized OCP: linearise -> Riccati LQ solve -> dual update ->
 * filter line search (same rule and grid as the single-robot step) -> update.  stats[5] as
 * oracle_srbd_step.  dirs optional. */
int oracle_multi_step(const oracle_srbd_params *P, const oracle_multi_params *M, int N, int n_alpha, double c1,
                      double theta_max, double *x, double *u, double *lam, const double *x0, const double *xref,
                      const double *uref, const uint8_t *contact, const double *feet, double *stats,
                      double *dx_out, double *du_out, double *dlam_out) {
    const int n = 12 * M->n_robots, m = n;
    const size_t S1 = (size_t)(N + 1), nn = (size_t)n * n;
    double *A = malloc(sizeof(double) * S1 * nn), *Bm = malloc(sizeof(double) * S1 * nn);
    double *c = malloc(sizeof(double) * S1 * n), *Q = malloc(sizeof(double) * S1 * nn);
    double *R = malloc(sizeof(double) * S1 * nn), *S = malloc(sizeof(double) * S1 * nn);
    double *q = malloc(sizeof(double) * S1 * n), *r = malloc(sizeof(double) * S1 * m);
    double *Pt = malloc(sizeof(double) * nn), *pt = malloc(sizeof(double) * n), *d0 = malloc(sizeof(double) * n);
    double *dx = malloc(sizeof(double) * (S1 + 1) * n), *du = malloc(sizeof(double) * S1 * m);
    double *dl = malloc(sizeof(double) * (S1 + 1) * n);
    double *xa = malloc(sizeof(double) * (S1 + 1) * n), *ua = malloc(sizeof(double) * S1 * m);
    double thr = theta_max > 0 ? theta_max : 1e-2 * (N + 1);
    int info = oracle_multi_linearize(P, M, N, x, u, lam, x0, xref, uref, contact, feet, A, Bm, c, Q, R, S, q, r,
                                      Pt, pt, d0);
    if (info == 0) info = oracle_solve_lq(N, n, m, A, Bm, c, Q, R, S, q, r, Pt, pt, d0, dx, du, dl, NULL, NULL, NULL, NULL);
    if (info == 0) {
        for (size_t t = 0; t < (S1 + 1) * n; ++t)
            if (!isfinite(dx[t]) || !isfinite(dl[t])) info = -1;
        for (size_t t = 0; t < S1 * m; ++t)
            if (!isfinite(du[t])) info = -1;
    }
    double J0 = oracle_multi_cost(P, M, N, x, u, xref, uref, contact);
    double th0 = oracle_multi_theta(P, M, N, x, u, x0, contact, feet);
    double alpha = 0, Jn = J0, thn = th0;
    int accepted = 0;
    if (info == 0) {
        double g = oracle_multi_cost_slope(P, M, N, x, u, xref, uref, contact, dx, du);
        for (int j = 0; j < n_alpha && !accepted; ++j) {
            double al = ldexp(1.0, -j);
            int ok = 1;
            for (size_t t = 0; t < (S1 + 1) * n; ++t) xa[t] = x[t] + al * dx[t];
            for (size_t t = 0; t < S1 * m; ++t) ua[t] = u[t] + al * du[t];
            for (int i = 0; i <= N; ++i)
                for (int k = 0; k < M->n_robots; ++k) ok &= pitch_ok(xa + (size_t)i * n + 12 * k);
            double Ja = ok ? oracle_multi_cost(P, M, N, xa, ua, xref, uref, contact) : INFINITY;
            double tha = ok ? oracle_multi_theta(P, M, N, xa, ua, x0, contact, feet) : INFINITY;
            if (filter_accept(J0, th0, g, Ja, tha, al, c1, thr)) {
                alpha = al; accepted = 1; Jn = Ja; thn = tha;
            }
        }
        if (accepted) {
            for (size_t t = 0; t < (S1 + 1) * n; ++t) { x[t] += alpha * dx[t]; lam[t] += alpha * dl[t]; }
            for (size_t t = 0; t < S1 * m; ++t) u[t] += alpha * du[t];
        }
    }
    if (stats) { stats[0] = Jn; stats[1] = thn; stats[2] = alpha; stats[3] = accepted; stats[4] = info; }
    if (dx_out) memcpy(dx_out, dx, sizeof(double) * (S1 + 1) * n);
    if (du_out) memcpy(du_out, du, sizeof(double) * S1 * m);
    if (dlam_out) memcpy(dlam_out, dl, sizeof(double) * (S1 + 1) * n);
    free(A); free(Bm); free(c); free(Q); free(R); free(S); free(q); free(r); free(Pt); free(pt); free(d0);
    free(dx); free(du); free(dl); free(xa); free(ua);
    return info;
}

/* Closed-loop plant ("plant = RK4 integration of the same SRBD model";
 * P:388 push disturbance): classical RK4 of xdot = f(x,u) + (0,0,0, 0,0,0, F_ext/m, 0,0,0),
 * `sub` steps of h = dt/sub, u / feet / contact held constant (zero-order hold).            */
void oracle_srbd_plant(const oracle_srbd_params *P, const double *x0, const double *u,
                       const double *feet, const uint8_t *contact, const double *F_ext /* [3] or NULL */,
                       double dt, int sub, double *x_out) {
    double x[NX], k1[NX], k2[NX], k3[NX], k4[NX], y[NX];
    memcpy(x, x0, sizeof x);
    const double h = dt / sub;
    for (int s = 0; s < sub; ++s) {
        oracle_srbd_f(P, x, u, feet, contact, k1);
        if (F_ext) for (int a = 0; a < 3; ++a) k1[6 + a] += F_ext[a] / P->mass;
        for (int r = 0; r < NX; ++r) y[r] = x[r] + 0.5 * h * k1[r];
        oracle_srbd_f(P, y, u, feet, contact, k2);
        if (F_ext) for (int a = 0; a < 3; ++a) k2[6 + a] += F_ext[a] / P->mass;
        for (int r = 0; r < NX; ++r) y[r] = x[r] + 0.5 * h * k2[r];
        oracle_srbd_f(P, y, u, feet, contact, k3);
        if (F_ext) for (int a = 0; a < 3; ++a) k3[6 + a] += F_ext[a] / P->mass;
        for (int r = 0; r < NX; ++r) y[r] = x[r] + h * k3[r];
        oracle_srbd_f(P, y, u, feet, contact, k4);
        if (F_ext) for (int a = 0; a < 3; ++a) k4[6 + a] += F_ext[a] / P->mass;
        for (int r = 0; r < NX; ++r) x[r] += h / 6.0 * (k1[r] + 2.0 * k2[r] + 2.0 * k3[r] + k4[r]);
    }
    memcpy(x_out, x, sizeof x);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
