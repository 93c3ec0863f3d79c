// srbd.cuh -- built-in single-rigid-body quadruped model on sm_100a:
//   k_srbd_linearize  A, B, b, Q, R, S, q, r, P_{N+1}, p_{N+1}, dx0 per stage (P:142-163,
//                     P:290-313); one worker per (instance, stage), lane r computes row r
//   k_srbd_linesearch filter line search on the fixed grid alpha = 2^-j, the linear
//                     update (Eq. 16) and the stats; one warp per instance, lanes over stages
// State x = [p, Theta = (roll, pitch, yaw) ZYX, v (world), w (body)], u = 4 world-frame GRFs.
// Explicit Euler h = x + dt f (reading R14); pitch guard |pitch| < pi/2 - 0.1 (reading R13).
#pragma once

#include "common.cuh"
#include "lq.cuh"

namespace pdilqr {

struct SrbdConst {
    double dt, mass, I[9], Iinv[9], g[3];
    double wx[12], wxt[12], wu_st, wu_sw;
    double mu, fmin, fmax, bmu, bdelta;
    double imass, ibd, ibd2;  // 1 / mass, 1 / bdelta, 1 / bdelta^2 (host-computed)
    double theta_max, c1;
    int n_alpha;
};

constexpr double kPitchGuard = 1.5707963267948966 - 0.1;

// relaxed barrier, feasible <=> xi > 0 (reading R11)
template <typename T>
__device__ __forceinline__ T barrier_val(T xi, T mu, T d) {
    if (xi >= d) return -mu * log(xi);
    const T t = (xi - T(2) * d) / d;
    return T(0.5) * mu * (t * t - T(1)) - mu * log(d);
}
template <typename T>
__device__ __forceinline__ T barrier_d1(T xi, T mu, T d) { return xi >= d ? -mu / xi : mu * (xi - T(2) * d) / (d * d); }
template <typename T>
__device__ __forceinline__ T barrier_d2(T xi, T mu, T d) { return xi >= d ? mu / (xi * xi) : mu / (d * d); }

// Barrier first and second derivatives with one reciprocal instead of IEEE divisions:
// xi >= d: (-mu / xi, mu / xi^2); else (mu (xi - 2 d) / d^2, mu / d^2), id2 = 1 / d^2.
template <typename T>
__device__ __forceinline__ void barrier_d12(T xi, T mu, T d, T id2, T &d1, T &d2) {
    const T rx = rcp_rn(xi);
    const bool in = xi >= d;
    d1 = in ? -mu * rx : mu * (xi - T(2) * d) * id2;
    d2 = in ? mu * rx * rx : mu * id2;
}

// Gradient and Hessian of the six friction-pyramid / normal-force barriers of one stance foot
// with respect to its force (fx, fy, fz), the constraint normals being constants:
//   grad = sum_c B'(xi_c) g_c,  H = sum_c B''(xi_c) g_c g_c^T  (H_xy = 0).
template <typename T>
struct FootBarrier {
    T gx, gy, gz, hxx, hyy, hzz, hxz, hyz;
};
template <typename T>
__device__ __forceinline__ FootBarrier<T> foot_barrier(const SrbdConst &K, T fx, T fy, T fz) {
    const T mu = T(K.mu), bmu = T(K.bmu), d = T(K.bdelta), id2 = T(K.ibd2);
    const T mfz = mu * fz;
    T a0, a1, a2, a3, a4, a5, b0, b1, b2, b3, b4, b5;
    barrier_d12<T>(mfz - fx, bmu, d, id2, a0, b0);
    barrier_d12<T>(mfz + fx, bmu, d, id2, a1, b1);
    barrier_d12<T>(mfz - fy, bmu, d, id2, a2, b2);
    barrier_d12<T>(mfz + fy, bmu, d, id2, a3, b3);
    barrier_d12<T>(fz - T(K.fmin), bmu, d, id2, a4, b4);
    barrier_d12<T>(T(K.fmax) - fz, bmu, d, id2, a5, b5);
    FootBarrier<T> o;
    o.gx = a1 - a0;
    o.gy = a3 - a2;
    o.gz = mu * ((a0 + a1) + (a2 + a3)) + (a4 - a5);
    o.hxx = b0 + b1;
    o.hyy = b2 + b3;
    o.hzz = mu * mu * ((b0 + b1) + (b2 + b3)) + (b4 + b5);
    o.hxz = mu * (b1 - b0);
    o.hyz = mu * (b3 - b2);
    return o;
}

// constraint c in 0..5 of one stance foot: xi = gx fx + gy fy + gz fz + h
//   0: mu fz - fx   1: mu fz + fx   2: mu fz - fy   3: mu fz + fy   4: fz - fmin   5: fmax - fz
template <typename T>
__device__ __forceinline__ void foot_con(int c, T mu, T fmin, T fmax, T &gx, T &gy, T &gz, T &h) {
    gx = (c == 0) ? T(-1) : (c == 1) ? T(1) : T(0);
    gy = (c == 2) ? T(-1) : (c == 3) ? T(1) : T(0);
    gz = (c < 4) ? mu : (c == 4) ? T(1) : T(-1);
    h = (c == 4) ? -fmin : (c == 5) ? fmax : T(0);
}

// sin / cos of the Euler angles in the linearisation: fp32 uses the SFU approximation (absolute
// error ~2^-21, below the fp32 rounding of the Jacobian entries it feeds); fp64 stays accurate.
__device__ __forceinline__ void lin_sincos(float x, float *s, float *c) { __sincosf(x, s, c); }
__device__ __forceinline__ void lin_sincos(double x, double *s, double *c) { sincos(x, s, c); }

// Continuous dynamics f(x,u) for one component index r (all lanes may call with their own r).
// Shared trig / rotation terms are recomputed per call (cheap, no smem traffic).
template <typename T>
struct SrbdEval {
    T sr, cr, sp, cp, sy, cy, tp, icp;
    T R[9];      // body -> world, R = Rz(yaw) Ry(pitch) Rx(roll)
    T tau[3];    // world torque sum_j c_j (r_j - p) x f_j
    T F[3];      // sum_j c_j f_j

    __device__ __forceinline__ void init(const SrbdConst &K, const T *x, const T *u, const T *feet, const uint8_t *con) {
        lin_sincos(x[3], &sr, &cr);
        lin_sincos(x[4], &sp, &cp);
        lin_sincos(x[5], &sy, &cy);
        icp = rcp_rn(cp);
        tp = sp * icp;
        R[0] = cy * cp; R[1] = cy * sp * sr - sy * cr; R[2] = cy * sp * cr + sy * sr;
        R[3] = sy * cp; R[4] = sy * sp * sr + cy * cr; R[5] = sy * sp * cr - cy * sr;
        R[6] = -sp;     R[7] = cp * sr;                R[8] = cp * cr;
        tau[0] = tau[1] = tau[2] = T(0);
        F[0] = F[1] = F[2] = T(0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!con[j]) continue;
            const T fx = u[3 * j], fy = u[3 * j + 1], fz = u[3 * j + 2];
            const T rx = feet[3 * j] - x[0], ry = feet[3 * j + 1] - x[1], rz = feet[3 * j + 2] - x[2];
            tau[0] += ry * fz - rz * fy;
            tau[1] += rz * fx - rx * fz;
            tau[2] += rx * fy - ry * fx;
            F[0] += fx; F[1] += fy; F[2] += fz;
        }
    }
    // wdot (body angular acceleration) component a
    __device__ __forceinline__ T wdot(const SrbdConst &K, const T *x, int a) const {
        const T w0 = x[9], w1 = x[10], w2 = x[11];
        T Iw[3], rhs[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) Iw[c] = T(K.I[3 * c]) * w0 + T(K.I[3 * c + 1]) * w1 + T(K.I[3 * c + 2]) * w2;
        const T wxIw[3] = {w1 * Iw[2] - w2 * Iw[1], w2 * Iw[0] - w0 * Iw[2], w0 * Iw[1] - w1 * Iw[0]};
#pragma unroll
        for (int c = 0; c < 3; ++c) rhs[c] = R[c] * tau[0] + R[3 + c] * tau[1] + R[6 + c] * tau[2] - wxIw[c];
        return T(K.Iinv[3 * a]) * rhs[0] + T(K.Iinv[3 * a + 1]) * rhs[1] + T(K.Iinv[3 * a + 2]) * rhs[2];
    }
    __device__ __forceinline__ T f(const SrbdConst &K, const T *x, int r) const {
        if (r < 3) return x[6 + r];
        if (r == 3) return x[9] + sr * tp * x[10] + cr * tp * x[11];
        if (r == 4) return cr * x[10] - sr * x[11];
        if (r == 5) return (sr * x[10] + cr * x[11]) * icp;
        if (r < 9) return F[r - 6] * T(K.imass) + T(K.g[r - 6]);
        return wdot(K, x, r - 9);
    }
    // all twelve components, the angular acceleration evaluated once
    __device__ __forceinline__ void f_all(const SrbdConst &K, const T *x, T (&out)[12]) const {
        const T w0 = x[9], w1 = x[10], w2 = x[11];
        out[0] = x[6]; out[1] = x[7]; out[2] = x[8];
        out[3] = w0 + sr * tp * w1 + cr * tp * w2;
        out[4] = cr * w1 - sr * w2;
        out[5] = (sr * w1 + cr * w2) * icp;
#pragma unroll
        for (int c = 0; c < 3; ++c) out[6 + c] = F[c] * T(K.imass) + T(K.g[c]);
        T Iw[3], rhs[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) Iw[c] = T(K.I[3 * c]) * w0 + T(K.I[3 * c + 1]) * w1 + T(K.I[3 * c + 2]) * w2;
        const T wxIw[3] = {w1 * Iw[2] - w2 * Iw[1], w2 * Iw[0] - w0 * Iw[2], w0 * Iw[1] - w1 * Iw[0]};
#pragma unroll
        for (int c = 0; c < 3; ++c) rhs[c] = R[c] * tau[0] + R[3 + c] * tau[1] + R[6 + c] * tau[2] - wxIw[c];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            out[9 + a] = T(K.Iinv[3 * a]) * rhs[0] + T(K.Iinv[3 * a + 1]) * rhs[1] + T(K.Iinv[3 * a + 2]) * rhs[2];
    }
};

// Row r of the stage-i linearisation computed by one lane:
//   Arow = dt Fx[r, :] (A = I + dt Fx; the identity is added by the caller), Brow = dt Fu[r, :],
//   fr = f_r(x, u), Rrow = row r of R = W_u + sum_c B''(xi_c) grad xi_c grad xi_c^T (control row r),
//   rg = W_u (u - uref)_r + sum_c B'(xi_c) grad xi_c[r]  (r_i without the multiplier term),
//   bad = outside the pitch guard or non-finite.
template <typename T>
struct SrbdRow {
    T Arow[12], Brow[12], Rrow[12];
    T fr, rg;
    bool bad;
};

template <typename T>
__device__ __forceinline__ void srbd_stage_row(const SrbdConst &K, const T *x, const T *u, const T *feet,
                                               const uint8_t *con, const T *ur, int r, SrbdRow<T> &o,
                                               T rho = T(0)) {
    constexpr int NX = 12;
    T xv[NX], uv[NX];
    ld_row<T, NX, true>(xv, x);
    ld_row<T, NX, true>(uv, u);
    SrbdEval<T> ev;
    ev.init(K, xv, uv, feet, con);
    const T dt = T(K.dt);
    T (&Arow)[NX] = o.Arow;
    T (&Brow)[NX] = o.Brow;
    zero(Arow); zero(Brow);
    const T w0 = xv[9], w1 = xv[10], w2 = xv[11];
    if (r < 3) {
#pragma unroll
        for (int c = 0; c < 3; ++c) Arow[6 + c] = (c == r) ? T(1) : T(0);
    } else if (r == 3) {
        Arow[3] = ev.tp * (ev.cr * w1 - ev.sr * w2);
        Arow[4] = (ev.sr * w1 + ev.cr * w2) * (ev.icp * ev.icp);
        Arow[9] = T(1); Arow[10] = ev.sr * ev.tp; Arow[11] = ev.cr * ev.tp;
    } else if (r == 4) {
        Arow[3] = -ev.sr * w1 - ev.cr * w2;
        Arow[10] = ev.cr; Arow[11] = -ev.sr;
    } else if (r == 5) {
        Arow[3] = (ev.cr * w1 - ev.sr * w2) * ev.icp;
        Arow[4] = (ev.sr * w1 + ev.cr * w2) * ev.sp * (ev.icp * ev.icp);
        Arow[10] = ev.sr * ev.icp; Arow[11] = ev.cr * ev.icp;
    } else if (r < 9) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int c = 0; c < 3; ++c) Brow[3 * j + c] = (con[j] && c == r - 6) ? T(K.imass) : T(0);
    } else {
        const int a = r - 9;
        T Ii[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) Ii[c] = T(K.Iinv[3 * a + c]);
        // Ma[b] = (I^-1 R^T)[a][b] = sum_c Iinv[a][c] R[b][c]
        T Ma[3];
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) Ma[bb] = Ii[0] * ev.R[3 * bb] + Ii[1] * ev.R[3 * bb + 1] + Ii[2] * ev.R[3 * bb + 2];
        // d wdot / d p = I^-1 R^T sum_j c_j [f_j]x
        T SF[9] = {T(0), -ev.F[2], ev.F[1], ev.F[2], T(0), -ev.F[0], -ev.F[1], ev.F[0], T(0)};
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) Arow[cc] = Ma[0] * SF[cc] + Ma[1] * SF[3 + cc] + Ma[2] * SF[6 + cc];
        // d wdot / d Theta_k = I^-1 (dR/dTheta_k)^T tau
        const T *R = ev.R;
        const T t0 = ev.tau[0], t1 = ev.tau[1], t2 = ev.tau[2];
        // dR/droll: col0 = 0, col1 = R col2, col2 = -R col1
        T v0[3] = {T(0), R[2] * t0 + R[5] * t1 + R[8] * t2, -(R[1] * t0 + R[4] * t1 + R[7] * t2)};
        // dR/dpitch entries
        const T cy = ev.cy, sy = ev.sy, cp = ev.cp, sp = ev.sp, sr = ev.sr, cr = ev.cr;
        const T dP[9] = {-cy * sp, cy * cp * sr, cy * cp * cr, -sy * sp, sy * cp * sr, sy * cp * cr, -cp, -sp * sr, -sp * cr};
        T v1[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) v1[c] = dP[c] * t0 + dP[3 + c] * t1 + dP[6 + c] * t2;
        // dR/dyaw: row0 = -R row1, row1 = R row0, row2 = 0
        T v2[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) v2[c] = -R[3 + c] * t0 + R[c] * t1;
        Arow[3] = Ii[0] * v0[0] + Ii[1] * v0[1] + Ii[2] * v0[2];
        Arow[4] = Ii[0] * v1[0] + Ii[1] * v1[1] + Ii[2] * v1[2];
        Arow[5] = Ii[0] * v2[0] + Ii[1] * v2[1] + Ii[2] * v2[2];
        // d wdot / d w = -I^-1 ([w]x I - [I w]x)
        T Iw[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) Iw[c] = T(K.I[3 * c]) * w0 + T(K.I[3 * c + 1]) * w1 + T(K.I[3 * c + 2]) * w2;
        const T Wx[9] = {T(0), -w2, w1, w2, T(0), -w0, -w1, w0, T(0)};
        const T IWx[9] = {T(0), -Iw[2], Iw[1], Iw[2], T(0), -Iw[0], -Iw[1], Iw[0], T(0)};
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            T s = T(0);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const T WI = Wx[3 * c] * T(K.I[cc]) + Wx[3 * c + 1] * T(K.I[3 + cc]) + Wx[3 * c + 2] * T(K.I[6 + cc]);
                s += Ii[c] * (WI - IWx[3 * c + cc]);
            }
            Arow[9 + cc] = -s;
        }
        // d wdot / d f_j = c_j I^-1 R^T [r_j - p]x
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!con[j]) continue;
            const T rx = feet[3 * j] - xv[0], ry = feet[3 * j + 1] - xv[1], rz = feet[3 * j + 2] - xv[2];
            const T Sr[9] = {T(0), -rz, ry, rz, T(0), -rx, -ry, rx, T(0)};
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) Brow[3 * j + cc] = Ma[0] * Sr[cc] + Ma[1] * Sr[3 + cc] + Ma[2] * Sr[6 + cc];
        }
    }
    T fr = T(0);
    {
        T fa[NX];
        ev.f_all(K, xv, fa);
#pragma unroll
        for (int c = 0; c < NX; ++c) fr = (c == r) ? fa[c] : fr;
    }
    // Arow holds dt Fx (the identity is added at the store): keeps A^T lam - lam = dt Fx^T lam
    // and the defect free of fp cancellation
#pragma unroll
    for (int j = 0; j < NX; ++j) { Arow[j] = dt * Arow[j]; Brow[j] = dt * Brow[j]; }
    const T ur_r = u[r];
    o.bad = !(fabs((double)xv[4]) < kPitchGuard) || !isfinite(fr) || !isfinite(x[r]) || !isfinite(ur_r);
    o.fr = fr;
    // control row r: foot j = r / 3, axis a = r % 3
    const int j = r / 3, a = r % 3;
    const bool stance = con[j] != 0;
    const T wu = stance ? T(K.wu_st) : T(K.wu_sw);
    T (&Rrow)[NX] = o.Rrow;
#pragma unroll
    for (int c = 0; c < NX; ++c) Rrow[c] = (c == r) ? wu + rho : T(0);   // rho: LM shift (pdilqr_solve)
    T rg = wu * (ur_r - (ur ? ur[r] : T(0)));
    {
        // barrier terms of this lane's foot j (stance only): gradient entry a, Hessian row a of the
        // foot's 3x3 block (columns 3j..3j+2)
        const FootBarrier<T> fb = foot_barrier<T>(K, uv[3 * j], uv[3 * j + 1], uv[3 * j + 2]);
        const T ga = a == 0 ? fb.gx : a == 1 ? fb.gy : fb.gz;
        const T h0 = a == 0 ? fb.hxx : a == 1 ? T(0) : fb.hxz;
        const T h1 = a == 0 ? T(0) : a == 1 ? fb.hyy : fb.hyz;
        const T h2 = a == 0 ? fb.hxz : a == 1 ? fb.hyz : fb.hzz;
        if (stance) rg += ga;
#pragma unroll
        for (int c = 0; c < NX; ++c) {
            const T hv = (c % 3 == 0) ? h0 : (c % 3 == 1) ? h1 : h2;
            Rrow[c] += (stance && c / 3 == j) ? hv : T(0);
        }
    }
    o.rg = rg;
}

// ------------------------------------------------------------------------- linearisation
// Lane r < 12 of the worker of stage i writes row r of A_i = I + dt Fx, B_i = dt Fu, Q_i, R_i,
// S_i (= 0), and b_i[r], q_i[r] (= W_x (x - xref) + A^T lam_{i+1} - lam_i), r_i[r]
// (= W_u (u - uref) + sum B'(xi) grad xi + B^T lam_{i+1}); the stage-(N+1) worker writes
// P_{N+1} = W_N, p_{N+1} = W_N (x_{N+1} - xref) - lam_{N+1} and dx0 = xhat0 - x_0.
template <typename T>
struct SrbdIter {
    const T *x, *u, *lam, *x0, *xref, *uref;
    const uint8_t *con;
    const T *feet;
    // pdilqr_solve bookkeeping (nullptr for a plain step): conv[b] = 0 active, k > 0 converged at
    // iteration k (frozen), -k stopped by a failure (info != 0) at iteration k; *active counts the
    // instances still active after this iteration.
    int32_t *conv = nullptr, *active = nullptr;
    double tol = 0.0;
    int iter = 0;
    // Levenberg-Marquardt ladder of pdilqr_solve (reading R28): rho[b] is added to every R_i of
    // instance b; the update kernel escalates it (0 -> 1e-6 -> ... -> 1e-2, x10) after a
    // factorisation failure or an all-rejected line search and resets it after an accepted step.
    double *rho = nullptr;
    __device__ __forceinline__ double rho_of(int b) const { return rho ? rho[b] : 0.0; }
};

constexpr double kLmRho0 = 1e-6, kLmRhoMax = 1e-2;

template <typename T>
__global__ void __launch_bounds__(128) k_srbd_linearize(SrbdConst K, SrbdIter<T> it, int B, int N, LqArgs<T> outc,
                                                        int32_t *pre_info) {
    constexpr int WS = 16, NX = 12;
    LqArgs<T> &o = outc;  // writable views (const-cast below)
    const int lane = worker_lane<WS>();
    const unsigned mask = worker_mask<WS>();
    const int wloc = threadIdx.x / WS;
    const long gw = (long)blockIdx.x * (blockDim.x / WS) + wloc;
    __shared__ __align__(16) T smA[8][NX * NX];
    __shared__ __align__(16) T smB[8][NX * NX];
    if (gw >= (long)B * (N + 2)) return;
    const int b = (int)(gw / (N + 2)), i = (int)(gw % (N + 2));
    const int r = lane < NX ? lane : 0;
    const T *x = it.x + ((size_t)b * (N + 2) + i) * NX;
    const T *lam = it.lam + ((size_t)b * (N + 2) + i) * NX;
    const T *xr = it.xref + ((size_t)b * (N + 2) + i) * NX;
    if (i == N + 1) {
        if (lane < NX) {
            T *Pt = const_cast<T *>(o.Pt) + (size_t)b * NX * NX + r * NX;
#pragma unroll
            for (int j = 0; j < NX; ++j) Pt[j] = (j == r) ? T(K.wxt[r]) : T(0);
            const_cast<T *>(o.pt)[(size_t)b * NX + r] = T(K.wxt[r]) * (x[r] - xr[r]) - lam[r];
            const T *x0 = it.x + (size_t)b * (N + 2) * NX;
            const_cast<T *>(o.dx0)[(size_t)b * NX + r] = it.x0[(size_t)b * NX + r] - x0[r];
            if (!isfinite(x[r]) || !isfinite(lam[r]) || !isfinite(it.x0[(size_t)b * NX + r])) pre_info[b] = -1;
        }
        return;
    }
    const size_t st = (size_t)b * (N + 1) + i;
    const T *u = it.u + st * NX;
    const T *feet = it.feet + st * 12;
    const uint8_t *con = it.con + st * 4;
    const T *ln = lam + NX;
    const T *ur = it.uref ? it.uref + st * NX : nullptr;
    SrbdRow<T> row;
    srbd_stage_row<T>(K, x, u, feet, con, ur, r, row, (T)it.rho_of(b));
    const T dt = T(K.dt);
    const T xr_r = x[r];
    const bool bad = row.bad || !isfinite(lam[r]);
    if (lane < NX) {
        st_row<T, NX, true>(smA[wloc] + r * NX, row.Arow);
        st_row<T, NX, true>(smB[wloc] + r * NX, row.Brow);
    }
    __syncwarp(mask);
    // column r of dt Fx and of B against lam_{i+1}
    T ATl = T(0), BTl = T(0);
#pragma unroll
    for (int t = 0; t < NX; ++t) { ATl = fma(smA[wloc][t * NX + r], ln[t], ATl); BTl = fma(smB[wloc][t * NX + r], ln[t], BTl); }
    const T fr = row.fr, rg = row.rg;
    T (&Arow)[NX] = row.Arow;
    T (&Brow)[NX] = row.Brow;
    T (&Rrow)[NX] = row.Rrow;
    if (lane < NX) {
        T *Ao = const_cast<T *>(o.A) + st * NX * NX + r * NX;
        T *Bo = const_cast<T *>(o.Bm) + st * NX * NX + r * NX;
        T *Qo = const_cast<T *>(o.Q) + st * NX * NX + r * NX;
        T *Ro = const_cast<T *>(o.R) + st * NX * NX + r * NX;
        T *So = const_cast<T *>(o.S) + st * NX * NX + r * NX;
        T Ar[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) Ar[j] = (j == r ? T(1) : T(0)) + Arow[j];
        st_row<T, NX, true>(Ao, Ar);
        st_row<T, NX, true>(Bo, Brow);
        T Qrow[NX], Zr[NX];
#pragma unroll
        for (int c = 0; c < NX; ++c) { Qrow[c] = (c == r) ? T(K.wx[r]) : T(0); Zr[c] = T(0); }
        st_row<T, NX, true>(Qo, Qrow);
        st_row<T, NX, true>(Ro, Rrow);
        st_row<T, NX, true>(So, Zr);
        const T xnext = x[NX + r];
        // b = h(x_i,u_i) - x_{i+1} = (x_i - x_{i+1}) + dt f ;  q = W (x - xref) + (lam_{i+1} - lam_i) + dt Fx^T lam_{i+1}
        const_cast<T *>(o.c)[st * NX + r] = (xr_r - xnext) + dt * fr;
        const_cast<T *>(o.q)[st * NX + r] = T(K.wx[r]) * (xr_r - xr[r]) + ((ln[r] - lam[r]) + ATl);
        const_cast<T *>(o.r)[st * NX + r] = rg + BTl;
        if (bad) pre_info[b] = -1;
    }
}

// -------------------------------------------------------------------------- line search
// One warp per instance; lane l handles stages l, l+32, ... and evaluates, for every alpha on
// the grid, its stage's cost and defect at the trial point x + alpha dx, u + alpha du.
// Trial points and differences in fp64, model evaluations in the handle dtype, all sums in
// fp64 in a fixed order (deterministic).  Stage cost l_i, terminal cost, theta per Eq. 17
// (reading R9), slope g = grad J . (dx, du), acceptance per P:286-287 (reading R10, see
// DESIGN.md), largest accepted alpha.  Then x, u, lam += alpha (dx, du, dlam) in place.
template <typename T>
struct LsOut {
    T *cost, *theta, *alpha;
    int32_t *accepted, *info;
};

// Linear update (Eq. 16) x, u, lam += alpha (dx, du, dlam) of instance b by one warp (coalesced),
// the step statistics, and the pdilqr_solve convergence test (theta <= tol and
// ||alpha (dx, du)||_inf <= tol).  Instances frozen by an earlier convergence or failure are not updated and
// report the current iterate (alpha = 0, accepted = 0).
template <typename T>
__device__ __forceinline__ void commit_step(const SrbdIter<T> &it, const LsOut<T> &so, int b, int N, int lane, bool acc,
                                            T alpha, double J0, double th0, double Jb, double thb, int info,
                                            const T *Dx, const T *Du, const T *Dl, double gslope) {
    const bool frozen = it.conv && it.conv[b] != 0;
    double smax = 0.0;
    if (acc && !frozen) {
        T *xw = const_cast<T *>(it.x) + (size_t)b * (N + 2) * 12;
        T *uw = const_cast<T *>(it.u) + (size_t)b * (N + 1) * 12;
        T *lw = const_cast<T *>(it.lam) + (size_t)b * (N + 2) * 12;
        T sm = T(0);
        // batches of 8 elements per lane: all loads of a batch issued before its stores (the
        // iterate and the direction may alias as far as the compiler knows), so a long horizon
        // is not one L2 round trip per element
        constexpr int UB = 8;
        const int nx = (N + 2) * 12, nu = (N + 1) * 12;
        for (int t0 = lane; t0 < nx; t0 += 32 * UB) {
            T xv[UB], dv[UB], lv[UB], ev[UB];
#pragma unroll
            for (int k = 0; k < UB; ++k) {
                const int t = t0 + 32 * k;
                if (t < nx) { xv[k] = xw[t]; dv[k] = Dx[t]; lv[k] = lw[t]; ev[k] = Dl[t]; }
            }
#pragma unroll
            for (int k = 0; k < UB; ++k) {
                const int t = t0 + 32 * k;
                if (t < nx) {
                    const T sx = alpha * dv[k];
                    xw[t] = xv[k] + sx;
                    lw[t] = lv[k] + alpha * ev[k];
                    sm = fmax(sm, fabs(sx));
                }
            }
        }
        for (int t0 = lane; t0 < nu; t0 += 32 * UB) {
            T uv[UB], dv[UB];
#pragma unroll
            for (int k = 0; k < UB; ++k) {
                const int t = t0 + 32 * k;
                if (t < nu) { uv[k] = uw[t]; dv[k] = Du[t]; }
            }
#pragma unroll
            for (int k = 0; k < UB; ++k) {
                const int t = t0 + 32 * k;
                if (t < nu) {
                    const T su = alpha * dv[k];
                    uw[t] = uv[k] + su;
                    sm = fmax(sm, fabs(su));
                }
            }
        }
        smax = (double)sm;
    }
    if (it.conv) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, off));
    }
    if (lane == 0) {
        if (frozen) {
            so.cost[b] = (T)J0;
            so.theta[b] = (T)th0;
            so.alpha[b] = T(0);
            so.accepted[b] = 0;
        } else {
            so.cost[b] = (T)Jb;
            so.theta[b] = (T)thb;
            so.alpha[b] = alpha;
            so.accepted[b] = acc ? 1 : 0;
            bool lm_retry = false;
            if (it.rho) {   // LM ladder: escalate after a factorisation failure or an all-rejected search
                const double r0 = it.rho[b];
                const bool fixed = !acc && info == 0 && th0 <= it.tol && fabs(gslope) <= it.tol * fmax(1.0, fabs(J0));
                if (acc) {
                    it.rho[b] = 0.0;
                } else if ((info > 0 || (info == 0 && !fixed)) && r0 < kLmRhoMax) {
                    it.rho[b] = r0 == 0.0 ? kLmRho0 : fmin(10.0 * r0, kLmRhoMax);
                    lm_retry = true;
                }
            }
            if (it.conv) {
                if (lm_retry) atomicAdd(it.active, 1);
                else if (info != 0) it.conv[b] = -it.iter;
                // accepted: theta and ||alpha (dx, du)||_inf within tol; every alpha rejected: the
                // iterate is kept, and it is a fixed point iff theta <= tol and the linear model
                // predicts no decrease, |grad J . (dx, du)| <= tol max(1, |J|) (R24)
                else if (acc ? (thb <= it.tol && smax <= it.tol)
                             : (th0 <= it.tol && fabs(gslope) <= it.tol * fmax(1.0, fabs(J0))))
                    it.conv[b] = it.iter;
                else atomicAdd(it.active, 1);
            }
        }
        so.info[b] = info;
    }
}

template <typename T>
__device__ __forceinline__ double stage_eval(const SrbdConst &K, const T *x, const T *dx, const T *xn, const T *dxn,
                                             const T *u, const T *du, const T *xr, const T *ur, const T *feet,
                                             const uint8_t *con, double alpha, double &defect2, bool &guard) {
    double xa[12], ua[12];
    T xs[12], us[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        xa[k] = (double)x[k] + alpha * (double)dx[k];
        ua[k] = (double)u[k] + alpha * (double)du[k];
        xs[k] = (T)xa[k];
        us[k] = (T)ua[k];
    }
    guard = guard || !(fabs(xa[4]) < kPitchGuard);
    double J = 0;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const double e = xa[k] - (double)xr[k];
        J += 0.5 * K.wx[k] * e * e;
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const double e = ua[k] - (ur ? (double)ur[k] : 0.0);
        J += 0.5 * (con[k / 3] ? K.wu_st : K.wu_sw) * e * e;
    }
    for (int j = 0; j < 4; ++j) {
        if (!con[j]) continue;
        for (int c = 0; c < 6; ++c) {
            T gx, gy, gz, h;
            foot_con<T>(c, T(K.mu), T(K.fmin), T(K.fmax), gx, gy, gz, h);
            const T xi = gx * us[3 * j] + gy * us[3 * j + 1] + gz * us[3 * j + 2] + h;
            J += (double)barrier_val<T>(xi, T(K.bmu), T(K.bdelta));
        }
    }
    SrbdEval<T> ev;
    ev.init(K, xs, us, feet, con);
    double d2 = 0;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const double d = ((double)xn[k] + alpha * (double)dxn[k]) - xa[k] - K.dt * (double)ev.f(K, xs, k);
        d2 += d * d;
    }
    defect2 = d2;
    return J;
}

// Lane map: lane l < 2*(na+1): alpha slot a = l % (na+1) (a = 0 is the current iterate,
// a >= 1 is alpha = 2^-(a-1)), stage group q = l / (na+1) (stages q, q+2, ...).  Each lane
// accumulates its J and theta in fp64 scalars; the two groups are added in a fixed order.
template <typename T>
__global__ void __launch_bounds__(128) k_srbd_linesearch(SrbdConst K, SrbdIter<T> it, int B, int N, const T *dx,
                                                         const T *du, const T *dlam, const int32_t *info_in,
                                                         LsOut<T> so) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (b >= B) return;
    const int na = K.n_alpha;          // <= 15
    const int ns = na + 1;
    const int a = lane % ns, q = lane / ns;
    const bool act = lane < 2 * ns;
    const double al = a == 0 ? 0.0 : ldexp(1.0, -(a - 1));
    const T *x = it.x + (size_t)b * (N + 2) * 12, *u = it.u + (size_t)b * (N + 1) * 12;
    const T *Dx = dx + (size_t)b * (N + 2) * 12, *Du = du + (size_t)b * (N + 1) * 12;
    const T *xr = it.xref + (size_t)b * (N + 2) * 12;
    const T *urf = it.uref ? it.uref + (size_t)b * (N + 1) * 12 : nullptr;
    const T *x0 = it.x0 + (size_t)b * 12;
    double J = 0, th = 0, g = 0;
    bool guard = false;
    if (act) {
        for (int i = q; i <= N; i += 2) {
            const T *xi = x + (size_t)i * 12, *dxi = Dx + (size_t)i * 12;
            const T *ui = u + (size_t)i * 12, *dui = Du + (size_t)i * 12;
            const T *feet = it.feet + ((size_t)b * (N + 1) + i) * 12;
            const uint8_t *con = it.con + ((size_t)b * (N + 1) + i) * 4;
            const T *uri = urf ? urf + (size_t)i * 12 : nullptr;
            double d2;
            J += stage_eval<T>(K, xi, dxi, xi + 12, dxi + 12, ui, dui, xr + (size_t)i * 12, uri, feet, con, al, d2, guard);
            th += sqrt(d2);
            if (a == 0) {  // slope of the cost at the current iterate (barriers included)
#pragma unroll
                for (int k = 0; k < 12; ++k) {
                    g += K.wx[k] * ((double)xi[k] - (double)xr[(size_t)i * 12 + k]) * (double)dxi[k];
                    g += (con[k / 3] ? K.wu_st : K.wu_sw) * ((double)ui[k] - (uri ? (double)uri[k] : 0.0)) * (double)dui[k];
                }
                for (int jf = 0; jf < 4; ++jf) {
                    if (!con[jf]) continue;
                    for (int c = 0; c < 6; ++c) {
                        T gx, gy, gz, h;
                        foot_con<T>(c, T(K.mu), T(K.fmin), T(K.fmax), gx, gy, gz, h);
                        const T xi_c = gx * ui[3 * jf] + gy * ui[3 * jf + 1] + gz * ui[3 * jf + 2] + h;
                        const double d1 = (double)barrier_d1<T>(xi_c, T(K.bmu), T(K.bdelta));
                        g += d1 * ((double)gx * dui[3 * jf] + (double)gy * dui[3 * jf + 1] + (double)gz * dui[3 * jf + 2]);
                    }
                }
            }
        }
        if (q == 0) {  // terminal cost and initial-condition term of theta (group 0 only)
            const T *xt = x + (size_t)(N + 1) * 12, *dxt = Dx + (size_t)(N + 1) * 12;
            double d0 = 0;
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                const double e = (double)xt[k] + al * (double)dxt[k] - (double)xr[(size_t)(N + 1) * 12 + k];
                J += 0.5 * K.wxt[k] * e * e;
                const double e0 = (double)x0[k] - ((double)x[k] + al * (double)Dx[k]);
                d0 += e0 * e0;
                if (a == 0) g += K.wxt[k] * ((double)xt[k] - (double)xr[(size_t)(N + 1) * 12 + k]) * (double)dxt[k];
            }
            th += sqrt(d0);
        }
    }
    // group 1 -> group 0 (fixed order: group0 + group1)
    const int src = (lane + ns) & 31;
    const double J1 = __shfl_sync(0xffffffffu, J, src), th1 = __shfl_sync(0xffffffffu, th, src);
    const double g1 = __shfl_sync(0xffffffffu, g, src);
    const int gd1 = __shfl_sync(0xffffffffu, (int)guard, src);
    J += J1; th += th1; g += g1; guard = guard || gd1;
    const double J0 = __shfl_sync(0xffffffffu, J, 0), th0 = __shfl_sync(0xffffffffu, th, 0);
    const double g0 = __shfl_sync(0xffffffffu, g, 0);
    const int info = info_in[b];
    bool ok = false;
    if (lane >= 1 && lane < ns && info == 0) {
        ok = !guard && isfinite(J) && isfinite(th);
        if (ok) {
            if (th0 > K.theta_max) ok = th <= th0;            // "reject if it further increases theta"
            else if (g0 < 0) ok = J <= J0 + K.c1 * al * g0;    // Armijo on descent directions
            else ok = (J < J0) || (th < th0);                   // cost or theta must decrease
        }
    }
    const unsigned acc = __ballot_sync(0xffffffffu, ok);
    const int jb = acc ? __ffs(acc) - 1 : 0;                   // smallest slot = largest alpha
    const double Jb = __shfl_sync(0xffffffffu, J, jb), thb = __shfl_sync(0xffffffffu, th, jb);
    const T alpha = acc ? (T)ldexp(1.0, -(jb - 1)) : T(0);
    commit_step<T>(it, so, b, N, lane, acc != 0u, alpha, J0, th0, Jb, thb, info, Dx, Du, dlam + (size_t)b * (N + 2) * 12, g0);
}

}  // namespace pdilqr
