// multi.cuh -- centralized multi-robot SRBD model (NEXT-3 of SURVEY §8(f); the paper's centralized
// controller for up to 16 quadrupeds):
//   state x = [x_robot0 (12) .. x_robot{R-1}], u likewise (n = m = 12 R); per robot the SRBD model and
//   cost of srbd.cuh; coupling by a collision-avoidance penalty 1/2 w eps^2 per robot pair and node,
//   eps = softplus_k(d_min - d), d = sqrt(|p_a - p_b|_xy^2 + eta^2) ("a quadratic penalty
//   term"), Gauss-Newton Hessian w grad eps grad eps^T.
//   k_multi_linearize  dense Eq. 4 blocks of one (instance, node) per CTA: block-diagonal robot
//                      linearisations (one 16-lane worker per robot, srbd_stage_row) + the pair
//                      terms (deterministic: one thread per position entry, pairs in fixed order)
//   k_multi_linesearch one CTA per instance: J(alpha), theta(alpha) on the alpha grid (threads over
//                      (node group, alpha slot), robots and pairs looped in fixed order, fp64 sums),
//                      the filter rule (reading R10), the update (Eq. 16) and the stats.
#pragma once

#include "srbd.cuh"

namespace pdilqr {

struct MultiConst {
    int R;                 // robots
    double d_min, w, k;    // collision distance, weight, softplus sharpness
};

constexpr double kCollEta = 1e-3;

// eps and grad eps w.r.t. (pa_x, pa_y, pb_x, pb_y) of one pair (fp64)
__device__ __forceinline__ double coll_pair(const MultiConst &M, double pax, double pay, double pbx, double pby,
                                            double (&g4)[4]) {
    const double dx = pax - pbx, dy = pay - pby;
    const double d = sqrt(dx * dx + dy * dy + kCollEta * kCollEta);
    const double s = M.k * (M.d_min - d);
    const double eps = (s > 0 ? s + log1p(exp(-s)) : log1p(exp(s))) / M.k;
    const double sig = 1.0 / (1.0 + exp(-s));
    g4[0] = -sig * dx / d; g4[1] = -sig * dy / d;
    g4[2] = sig * dx / d;  g4[3] = sig * dy / d;
    return eps;
}

__device__ __forceinline__ void pair_of(int p, int R, int &a, int &b) {  // p-th pair (a < b), row-major
    a = 0;
    int rem = p;
    while (rem >= R - 1 - a) { rem -= R - 1 - a; ++a; }
    b = a + 1 + rem;
}

constexpr int MULTI_THREADS = 256;
constexpr int MULTI_MAX_R = 21;   // n = 12 R <= 256
constexpr int MULTI_MAX_PAIRS = MULTI_MAX_R * (MULTI_MAX_R - 1) / 2;

// One CTA per (instance b, node i), i = 0..N+1.  Node N+1 writes P_{N+1}, p_{N+1}, dx0.
template <typename T>
__global__ void __launch_bounds__(MULTI_THREADS) k_multi_linearize(SrbdConst K, MultiConst M, SrbdIter<T> it, int B,
                                                                   int N, LqArgs<T> outc, int32_t *pre_info) {
    constexpr int WS = 16, NX = 12, NW = MULTI_THREADS / WS;
    __shared__ __align__(16) T smA[NW][NX * NX];
    __shared__ __align__(16) T smB[NW][NX * NX];
    __shared__ double s_eps[MULTI_MAX_PAIRS], s_g[MULTI_MAX_PAIRS][4];
    const int R = M.R, n = 12 * R;
    const int b = blockIdx.x / (N + 2), i = blockIdx.x % (N + 2);
    if (b >= B) return;
    const bool term = i == N + 1;
    const size_t nn = (size_t)n * n;
    const size_t st = (size_t)b * (N + 1) + (term ? 0 : i);
    T *Qo = const_cast<T *>(term ? outc.Pt + (size_t)b * nn : outc.Q + st * nn);
    T *qo = const_cast<T *>(term ? outc.pt + (size_t)b * n : outc.q + st * n);
    // phase 0: zero the dense blocks of this node
    {
        T *blk[5] = {Qo, nullptr, nullptr, nullptr, nullptr};
        int nb = 1;
        if (!term) {
            blk[1] = const_cast<T *>(outc.A) + st * nn;
            blk[2] = const_cast<T *>(outc.Bm) + st * nn;
            blk[3] = const_cast<T *>(outc.R) + st * nn;
            blk[4] = const_cast<T *>(outc.S) + st * nn;
            nb = 5;
        }
        for (int q = 0; q < nb; ++q)
            for (size_t t = threadIdx.x; t < nn; t += MULTI_THREADS) blk[q][t] = T(0);
    }
    __syncthreads();
    // phase 1: robot blocks (worker w = robot k, k = w, w + NW, ...)
    const int wk = threadIdx.x / WS, lane = threadIdx.x % WS;
    const unsigned wmask = 0xFFFFu << (threadIdx.x & 16);
    const int r = lane < NX ? lane : 0;
    for (int k0 = 0; k0 < R; k0 += NW) {
        const int k = k0 + wk;
        if (k < R) {
            const T *x = it.x + ((size_t)b * (N + 2) + i) * n + 12 * k;
            const T *lam = it.lam + ((size_t)b * (N + 2) + i) * n + 12 * k;
            const T *xr = it.xref + ((size_t)b * (N + 2) + i) * n + 12 * k;
            if (term) {
                if (lane < NX) {
                    T *P = Qo + (size_t)(12 * k + r) * n + 12 * k;
#pragma unroll
                    for (int j = 0; j < NX; ++j) P[j] = (j == r) ? T(K.wxt[r]) : T(0);
                    qo[12 * k + r] = T(K.wxt[r]) * (x[r] - xr[r]) - lam[r];
                    const T *xs = it.x + (size_t)b * (N + 2) * n + 12 * k;
                    const_cast<T *>(outc.dx0)[(size_t)b * n + 12 * k + r] = it.x0[(size_t)b * n + 12 * k + r] - xs[r];
                    if (!isfinite(x[r]) || !isfinite(lam[r]) || !isfinite(it.x0[(size_t)b * n + 12 * k + r])) pre_info[b] = -1;
                }
            } else {
                const T *u = it.u + st * n + 12 * k;
                const T *feet = it.feet + st * 12 * R + 12 * k;
                const uint8_t *con = it.con + st * 4 * R + 4 * k;
                const T *ln = lam + n;
                const T *ur = it.uref ? it.uref + st * n + 12 * k : nullptr;
                SrbdRow<T> row;
                srbd_stage_row<T>(K, x, u, feet, con, ur, r, row);
                const bool bad = row.bad || !isfinite(lam[r]);
                if (lane < NX) {
                    st_row<T, NX, true>(smA[wk] + r * NX, row.Arow);
                    st_row<T, NX, true>(smB[wk] + r * NX, row.Brow);
                }
                __syncwarp(wmask);
                T ATl = T(0), BTl = T(0);
#pragma unroll
                for (int t = 0; t < NX; ++t) { ATl = fma(smA[wk][t * NX + r], ln[t], ATl); BTl = fma(smB[wk][t * NX + r], ln[t], BTl); }
                if (lane < NX) {
                    const size_t ro = (size_t)(12 * k + r) * n + 12 * k;
                    T *Ao = const_cast<T *>(outc.A) + st * nn + ro;
                    T *Bo = const_cast<T *>(outc.Bm) + st * nn + ro;
                    T *Ro = const_cast<T *>(outc.R) + st * nn + ro;
#pragma unroll
                    for (int j = 0; j < NX; ++j) {
                        Ao[j] = (j == r ? T(1) : T(0)) + row.Arow[j];
                        Bo[j] = row.Brow[j];
                        Ro[j] = row.Rrow[j];
                    }
                    Qo[ro + r] = T(K.wx[r]);
                    const T xnext = x[n + r];
                    const_cast<T *>(outc.c)[st * n + 12 * k + r] = (x[r] - xnext) + T(K.dt) * row.fr;
                    qo[12 * k + r] = T(K.wx[r]) * (x[r] - xr[r]) + ((ln[r] - lam[r]) + ATl);
                    const_cast<T *>(outc.r)[st * n + 12 * k + r] = row.rg + BTl;
                    if (bad) pre_info[b] = -1;
                }
                __syncwarp(wmask);
            }
        }
    }
    // phase 2: collision pairs at this node
    const int np = R * (R - 1) / 2;
    const T *xn = it.x + ((size_t)b * (N + 2) + i) * n;
    for (int p = threadIdx.x; p < np; p += MULTI_THREADS) {
        int a, c;
        pair_of(p, R, a, c);
        double g4[4];
        s_eps[p] = coll_pair(M, (double)xn[12 * a], (double)xn[12 * a + 1], (double)xn[12 * c], (double)xn[12 * c + 1], g4);
#pragma unroll
        for (int s = 0; s < 4; ++s) s_g[p][s] = g4[s];
    }
    __syncthreads();
    // position entries (robot a, axis al) x (robot c, axis be): Q += w sum_p g g^T; q += w sum_p eps g
    for (int e = threadIdx.x; e < 4 * R * R; e += MULTI_THREADS) {
        const int a = e / (2 * R * 2), rem = e % (4 * R);
        const int al = (e / (2 * R)) % 2;
        const int c = (rem % (2 * R)) / 2, be = rem % 2;
        (void)rem;
        double v = 0;
        if (a == c) {
            for (int o = 0; o < R; ++o) {     // every pair containing robot a, in pair order
                if (o == a) continue;
                const int lo = min(a, o), hi = max(a, o);
                const int p = lo * (2 * R - lo - 1) / 2 + (hi - lo - 1);
                const int ia = (a == lo) ? al : 2 + al, ib = (a == lo) ? be : 2 + be;
                v += M.w * s_g[p][ia] * s_g[p][ib];
            }
        } else {
            const int lo = min(a, c), hi = max(a, c);
            const int p = lo * (2 * R - lo - 1) / 2 + (hi - lo - 1);
            const int ia = (a == lo) ? al : 2 + al, ib = (c == lo) ? be : 2 + be;
            v = M.w * s_g[p][ia] * s_g[p][ib];
        }
        if (v != 0) Qo[(size_t)(12 * a + al) * n + 12 * c + be] += T(v);
    }
    for (int e = threadIdx.x; e < 2 * R; e += MULTI_THREADS) {
        const int a = e / 2, al = e % 2;
        double v = 0;
        for (int o = 0; o < R; ++o) {
            if (o == a) continue;
            const int lo = min(a, o), hi = max(a, o);
            const int p = lo * (2 * R - lo - 1) / 2 + (hi - lo - 1);
            v += M.w * s_eps[p] * s_g[p][(a == lo) ? al : 2 + al];
        }
        qo[12 * a + al] += T(v);
    }
}

// Collision cost of one node at the trial positions x + alpha dx (fp64), and its slope at alpha = 0.
template <typename T>
__device__ __forceinline__ double node_coll(const MultiConst &M, const T *x, const T *dx, double al, double *slope) {
    double J = 0, g = 0;
    for (int a = 0; a < M.R; ++a)
        for (int c = a + 1; c < M.R; ++c) {
            double g4[4];
            const double pax = (double)x[12 * a] + al * (double)dx[12 * a], pay = (double)x[12 * a + 1] + al * (double)dx[12 * a + 1];
            const double pbx = (double)x[12 * c] + al * (double)dx[12 * c], pby = (double)x[12 * c + 1] + al * (double)dx[12 * c + 1];
            const double e = coll_pair(M, pax, pay, pbx, pby, g4);
            J += 0.5 * M.w * e * e;
            if (slope)
                g += M.w * e * (g4[0] * (double)dx[12 * a] + g4[1] * (double)dx[12 * a + 1] + g4[2] * (double)dx[12 * c] +
                                g4[3] * (double)dx[12 * c + 1]);
        }
    if (slope) *slope += g;
    return J;
}

// Filter line search + update, one CTA per instance.  Thread t: alpha slot a = t % ns (a = 0 the
// current iterate), node group q = t / ns (nodes q, q + G, ...).  Per node: every robot's stage
// cost and defect (stage_eval of srbd.cuh), theta adds |stacked defect|_2; collision terms on all
// nodes 0..N+1; terminal cost and the initial-condition defect in group 0.  Group partials are
// summed by thread a in group order (deterministic).
template <typename T>
__global__ void __launch_bounds__(MULTI_THREADS) k_multi_linesearch(SrbdConst K, MultiConst M, SrbdIter<T> it, int B,
                                                                    int N, const T *dx, const T *du, const T *dlam,
                                                                    const int32_t *info_lq, const int32_t *pre,
                                                                    LsOut<T> so) {
    __shared__ double sJ[MULTI_THREADS], sT[MULTI_THREADS], sG[MULTI_THREADS];
    __shared__ int sGd[MULTI_THREADS];
    __shared__ double fin[4];
    __shared__ int s_acc;
    __shared__ T s_alpha;
    const int b = blockIdx.x;
    if (b >= B) return;
    const int R = M.R, n = 12 * R;
    const int na = K.n_alpha, ns = na + 1, G = MULTI_THREADS / ns;
    const int t = threadIdx.x, a = t % ns, q = t / ns;
    const double al = a == 0 ? 0.0 : ldexp(1.0, -(a - 1));
    const T *x = it.x + (size_t)b * (N + 2) * n, *u = it.u + (size_t)b * (N + 1) * n;
    const T *Dx = dx + (size_t)b * (N + 2) * n, *Du = du + (size_t)b * (N + 1) * n;
    const T *xr = it.xref + (size_t)b * (N + 2) * n;
    const T *urf = it.uref ? it.uref + (size_t)b * (N + 1) * n : nullptr;
    double J = 0, th = 0, g = 0;
    bool guard = false;
    if (q < G) {
        for (int i = q; i <= N + 1; i += G) {
            const T *xi = x + (size_t)i * n, *dxi = Dx + (size_t)i * n;
            J += node_coll<T>(M, xi, dxi, al, a == 0 ? &g : nullptr);
            if (i == N + 1) continue;
            double d2s = 0;
            for (int k = 0; k < R; ++k) {
                const T *xk = xi + 12 * k, *dxk = dxi + 12 * k;
                const T *uk = u + (size_t)i * n + 12 * k, *duk = Du + (size_t)i * n + 12 * k;
                const T *feet = it.feet + ((size_t)b * (N + 1) + i) * 12 * R + 12 * k;
                const uint8_t *con = it.con + ((size_t)b * (N + 1) + i) * 4 * R + 4 * k;
                const T *urk = urf ? urf + (size_t)i * n + 12 * k : nullptr;
                const T *xrk = xr + (size_t)i * n + 12 * k;
                double d2;
                J += stage_eval<T>(K, xk, dxk, xk + n, dxk + n, uk, duk, xrk, urk, feet, con, al, d2, guard);
                d2s += d2;
                if (a == 0) {
#pragma unroll
                    for (int c = 0; c < 12; ++c) {
                        g += K.wx[c] * ((double)xk[c] - (double)xrk[c]) * (double)dxk[c];
                        g += (con[c / 3] ? K.wu_st : K.wu_sw) * ((double)uk[c] - (urk ? (double)urk[c] : 0.0)) * (double)duk[c];
                    }
                    for (int jf = 0; jf < 4; ++jf) {
                        if (!con[jf]) continue;
                        for (int c = 0; c < 6; ++c) {
                            T gx, gy, gz, h;
                            foot_con<T>(c, T(K.mu), T(K.fmin), T(K.fmax), gx, gy, gz, h);
                            const T xi_c = gx * uk[3 * jf] + gy * uk[3 * jf + 1] + gz * uk[3 * jf + 2] + h;
                            const double d1 = (double)barrier_d1<T>(xi_c, T(K.bmu), T(K.bdelta));
                            g += d1 * ((double)gx * duk[3 * jf] + (double)gy * duk[3 * jf + 1] + (double)gz * duk[3 * jf + 2]);
                        }
                    }
                }
            }
            th += sqrt(d2s);
        }
        if (q == 0) {   // terminal cost and the initial-condition term of theta
            const T *xt = x + (size_t)(N + 1) * n, *dxt = Dx + (size_t)(N + 1) * n;
            const T *x0 = it.x0 + (size_t)b * n;
            double d0 = 0;
            for (int c = 0; c < n; ++c) {
                const double e = (double)xt[c] + al * (double)dxt[c] - (double)xr[(size_t)(N + 1) * n + c];
                J += 0.5 * K.wxt[c % 12] * e * e;
                const double e0 = (double)x0[c] - ((double)x[c] + al * (double)Dx[c]);
                d0 += e0 * e0;
                if (a == 0) g += K.wxt[c % 12] * ((double)xt[c] - (double)xr[(size_t)(N + 1) * n + c]) * (double)dxt[c];
            }
            th += sqrt(d0);
        }
    }
    sJ[t] = J; sT[t] = th; sG[t] = g; sGd[t] = guard ? 1 : 0;
    __syncthreads();
    if (t < ns) {   // slot a = t: sum over the node groups in order
        double Js = 0, Ts = 0, gs = 0;
        int gd = 0;
        for (int qq = 0; qq < G; ++qq) {
            Js += sJ[qq * ns + t]; Ts += sT[qq * ns + t]; gd |= sGd[qq * ns + t];
            if (t == 0) gs += sG[qq * ns];
        }
        sJ[t] = Js; sT[t] = Ts; sGd[t] = gd;
        if (t == 0) fin[2] = gs;
    }
    __syncthreads();
    if (t == 0) {
        const int info = pre[b] != 0 ? pre[b] : info_lq[b];
        const double J0 = sJ[0], th0 = sT[0], g0 = fin[2];
        int jb = -1;
        if (info == 0) {
            for (int s = 1; s <= na && jb < 0; ++s) {
                const double Ja = sJ[s], tha = sT[s], als = ldexp(1.0, -(s - 1));
                bool ok = !sGd[s] && isfinite(Ja) && isfinite(tha);
                if (ok) {
                    if (th0 > K.theta_max) ok = tha <= th0;
                    else if (g0 < 0) ok = Ja <= J0 + K.c1 * als * g0;
                    else ok = (Ja < J0) || (tha < th0);
                }
                if (ok) jb = s;
            }
        }
        s_acc = jb;
        s_alpha = jb >= 0 ? (T)ldexp(1.0, -(jb - 1)) : T(0);
        so.cost[b] = (T)(jb >= 0 ? sJ[jb] : J0);
        so.theta[b] = (T)(jb >= 0 ? sT[jb] : th0);
        so.alpha[b] = s_alpha;
        so.accepted[b] = jb >= 0 ? 1 : 0;
        so.info[b] = info;
    }
    __syncthreads();
    if (s_acc >= 0) {   // x, u, lam += alpha (dx, du, dlam)  (Eq. 16)
        const T alpha = s_alpha;
        T *xw = const_cast<T *>(it.x) + (size_t)b * (N + 2) * n;
        T *uw = const_cast<T *>(it.u) + (size_t)b * (N + 1) * n;
        T *lw = const_cast<T *>(it.lam) + (size_t)b * (N + 2) * n;
        const T *Dl = dlam + (size_t)b * (N + 2) * n;
        for (size_t e = t; e < (size_t)(N + 2) * n; e += MULTI_THREADS) {
            xw[e] += alpha * Dx[e];
            lw[e] += alpha * Dl[e];
        }
        for (size_t e = t; e < (size_t)(N + 1) * n; e += MULTI_THREADS) uw[e] += alpha * Du[e];
    }
}

}  // namespace pdilqr
