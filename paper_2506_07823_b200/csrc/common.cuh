// common.cuh -- worker-level primitives for small dense matrix algebra on sm_100a.
//
// Execution model: a *worker* is a group of WS lanes of one warp
// (WS = 4, 8, 16 or 32, the next power of two >= max(n, m)).  Lane r of a worker owns ROW r of
// every matrix it computes on, held in registers with compile-time indices (fully unrolled
// loops, no local memory).  The other operand of a product is staged in the worker's private
// shared-memory slice and read with broadcast (all lanes of a worker read the same address;
// the two workers of a warp read two addresses in different banks) using 16-byte vector loads.
// Pivot rows of Gauss-Jordan eliminations travel by warp shuffles inside the worker.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pdilqr {

__host__ __device__ constexpr int worker_width(int d) { return d <= 4 ? 4 : d <= 8 ? 8 : d <= 16 ? 16 : 32; }
__host__ __device__ constexpr int round_up4(int d) { return (d + 3) & ~3; }

// --------------------------------------------------------------------------------- workers
// Lane mask of the calling thread's worker.  Workers of one warp may diverge (different loop
// trip counts), so every shuffle / __syncwarp uses the worker's own mask.
template <int WS>
__device__ __forceinline__ unsigned worker_mask() {
    if constexpr (WS == 32) return 0xffffffffu;
    else return ((1u << WS) - 1u) << (threadIdx.x & 31 & ~(WS - 1));
}
template <int WS>
__device__ __forceinline__ int worker_lane() { return threadIdx.x & (WS - 1); }

template <int WS, typename T>
__device__ __forceinline__ T wbcast(unsigned mask, T v, int src) { return __shfl_sync(mask, v, src, WS); }
template <int WS, typename T>
__device__ __forceinline__ T wxor(unsigned mask, T v, int m) { return __shfl_xor_sync(mask, v, m, WS); }

// ------------------------------------------------------------------------ vector row access
// Copy NC contiguous values src[0..NC) into registers.  Vectorised (16 B) when the compile-time
// shape allows it; `valid` < NC zero-fills the tail (padded instantiations).
template <typename T, int NC, bool VEC>
__device__ __forceinline__ void ld_row(T (&d)[NC], const T *__restrict__ s, int valid = NC) {
    if constexpr (VEC && sizeof(T) == 4 && NC % 4 == 0) {
#pragma unroll
        for (int j = 0; j < NC; j += 4) {
            float4 v = *reinterpret_cast<const float4 *>(s + j);
            d[j] = v.x; d[j + 1] = v.y; d[j + 2] = v.z; d[j + 3] = v.w;
        }
    } else if constexpr (VEC && sizeof(T) == 8 && NC % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NC; j += 2) {
            double2 v = *reinterpret_cast<const double2 *>(s + j);
            d[j] = v.x; d[j + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < NC; ++j) d[j] = (j < valid) ? s[j] : T(0);
    }
}

template <typename T, int NC, bool VEC>
__device__ __forceinline__ void st_row(T *__restrict__ d, const T (&s)[NC], int valid = NC) {
    if constexpr (VEC && sizeof(T) == 4 && NC % 4 == 0) {
#pragma unroll
        for (int j = 0; j < NC; j += 4) *reinterpret_cast<float4 *>(d + j) = make_float4(s[j], s[j + 1], s[j + 2], s[j + 3]);
    } else if constexpr (VEC && sizeof(T) == 8 && NC % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NC; j += 2) *reinterpret_cast<double2 *>(d + j) = make_double2(s[j], s[j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < NC; ++j)
            if (j < valid) d[j] = s[j];
    }
}

// Strided column load: d[k] = s[k * ld], k < valid (zero beyond).
template <typename T, int NK>
__device__ __forceinline__ void ld_col(T (&d)[NK], const T *__restrict__ s, int ld, int valid = NK) {
#pragma unroll
    for (int k = 0; k < NK; ++k) d[k] = (k < valid) ? s[k * ld] : T(0);
}

template <typename T, int NC>
__device__ __forceinline__ void zero(T (&d)[NC]) {
#pragma unroll
    for (int j = 0; j < NC; ++j) d[j] = T(0);
}

// -------------------------------------------------------------------- packed FP32 FMA (sm_100)
// c0 += a0*b0, c1 += a1*b1 as one FFMA2 (fma.rn.f32x2): halves the FMA instruction count of every
// row product; ptxas folds a broadcast scalar operand (a0 == a1) into the .F32 operand form.
__device__ __forceinline__ void ffma2(float a0, float a1, float b0, float b1, float &c0, float &c1) {
    asm("{\n .reg .b64 ra, rb, rc;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n mov.b64 rc, {%0, %1};\n"
        " fma.rn.f32x2 rc, ra, rb, rc;\n mov.b64 {%0, %1}, rc;\n}"
        : "+f"(c0), "+f"(c1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void ffma2(double a0, double a1, double b0, double b1, double &c0, double &c1) {
    c0 = fma(a0, b0, c0);
    c1 = fma(a1, b1, c1);
}

// ------------------------------------------------------------------------------ products
// out[j] (+)= sum_k a[k] * Y[k*LDY + j]   (row of a 1xK times KxNC matrix in shared memory)
template <typename T, int K, int NC, int LDY>
__device__ __forceinline__ void row_mat(T (&out)[NC], const T (&a)[K], const T *__restrict__ Y) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T y[NC];
        ld_row<T, NC, (LDY % (16 / sizeof(T)) == 0)>(y, Y + k * LDY);
        if constexpr (NC % 2 == 0) {
#pragma unroll
            for (int j = 0; j < NC; j += 2) ffma2(a[k], a[k], y[j], y[j + 1], out[j], out[j + 1]);
        } else {
#pragma unroll
            for (int j = 0; j < NC; ++j) out[j] = fma(a[k], y[j], out[j]);
        }
    }
}

// out[j] (+)= sum_k a[k] * Y[j*LDY + k]   (row times the transpose of an NCxK smem matrix)
template <typename T, int K, int NC, int LDY>
__device__ __forceinline__ void row_matT(T (&out)[NC], const T (&a)[K], const T *__restrict__ Y) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        T y[K];
        ld_row<T, K, (LDY % (16 / sizeof(T)) == 0)>(y, Y + j * LDY);
        if constexpr (K % 2 == 0) {
            T s0 = out[j], s1 = T(0);
#pragma unroll
            for (int k = 0; k < K; k += 2) ffma2(a[k], a[k + 1], y[k], y[k + 1], s0, s1);
            out[j] = s0 + s1;
        } else {
            T s = out[j];
#pragma unroll
            for (int k = 0; k < K; ++k) s = fma(a[k], y[k], s);
            out[j] = s;
        }
    }
}

// dot of a register row with a shared-memory vector
template <typename T, int K>
__device__ __forceinline__ T row_dot(const T (&a)[K], const T *__restrict__ v, T acc) {
    T y[K];
    ld_row<T, K, (K % (16 / sizeof(T)) == 0)>(y, v);
    if constexpr (K % 2 == 0) {
        T s1 = T(0);
#pragma unroll
        for (int k = 0; k < K; k += 2) ffma2(a[k], a[k + 1], y[k], y[k + 1], acc, s1);
        return acc + s1;
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) acc = fma(a[k], y[k], acc);
        return acc;
    }
}

// Branchless reciprocal for elimination multipliers: MUFU.RCP approximation refined by Newton
// steps (fp32: one step, <= 1 ulp; fp64: two steps).  No subnormal / slow-path handling: pivots
// are normal numbers (a zero or non-finite pivot is reported through the `ok` flag).
__device__ __forceinline__ float rcp_rn(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.0f), r);
}
__device__ __forceinline__ double rcp_rn(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}

// ------------------------------------------------------------------- Gauss-Jordan solves
// Solve  M X = RHS  for an NR x NR system distributed one row per lane (lane r < nrows owns
// row r of M in a[] and of RHS in rhs[]), in place.  Lanes r >= nrows are idle (never pivot).
//
// PIVOT = true : partial pivoting by implicit row selection (max |a[k]| over rows not yet used;
//                ties -> lowest lane).  Rows are never moved: on return the lane that pivoted
//                column k holds solution row k, and `piv_row` of every lane = the column it
//                pivoted (-1 for idle lanes).  Used for M = I + C~ P~ (nonsymmetric).
// PIVOT = false: no pivoting, pivot k = lane k; for symmetric positive definite M (R, G), where
//                every pivot is a ratio of leading principal minors and must be > 0.
// Returns false (uniformly across the worker) if a pivot is zero / non-finite (singular) or, for
// PIVOT = false, non-positive (not positive definite).
// FULLWARP = true: the caller guarantees the whole warp is converged and passes mask = all lanes
// (several workers per warp); the pivot search is then an xor butterfly inside each worker's
// WS-lane segment (plain SHFL.BFLY, no per-worker mask bookkeeping).
template <typename T, int WS, int NR, int NRHS, bool PIVOT, bool FULLWARP = false>
__device__ __forceinline__ bool gauss_jordan(unsigned mask, T (&a)[NR], T (&rhs)[NRHS], int lane, int nrows,
                                             int &piv_row) {
    // Unnormalised Gauss-Jordan: pivot rows are never scaled during the sweep (multiplier 0 on
    // the pivot lane, so every update is one shuffle + one FMA, no select); each pivot row is
    // divided by its pivot once at the end.  Same result as the normalised sweep in exact
    // arithmetic.
    bool used = lane >= nrows;
    bool ok = true;
    piv_row = -1;
    T mypiv = T(1);
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        if (k >= nrows) break;
        int p;
        if constexpr (PIVOT) {
            // one REDUX instead of a shuffle butterfly: key = |a| (fp32 bit pattern, monotonic for
            // non-negative values) with the low 5 bits replaced by (31 - lane): max key = largest
            // |a| among unused rows, ties -> lowest lane; NaN wins (then the pivot check fails).
            const float fa = fabsf((float)a[k]);
            const unsigned key = used ? 0u : ((__float_as_uint(fa) & 0xFFFFFFE0u) | (31u - (unsigned)lane));
            unsigned best;
            if constexpr (FULLWARP && WS == 32) {
                best = __reduce_max_sync(0xffffffffu, key);
            } else if constexpr (FULLWARP && WS == 16) {
                // two full-warp REDUX (one per half-warp worker), no per-worker mask bookkeeping
                const bool lo = (threadIdx.x & 16) == 0;
                const unsigned b0 = __reduce_max_sync(0xffffffffu, lo ? key : 0u);
                const unsigned b1 = __reduce_max_sync(0xffffffffu, lo ? 0u : key);
                best = lo ? b0 : b1;
            } else if constexpr (FULLWARP) {
                best = key;
#pragma unroll
                for (int off = WS / 2; off >= 1; off >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, off, WS));
            } else {
                best = __reduce_max_sync(mask, key);
            }
            p = 31 - (int)(best & 31u);
        } else {
            p = k;
        }
        // reciprocal computed speculatively by every lane, the pivot lane's value is broadcast
        const T rk = rcp_rn(a[k]);
        const T pv = wbcast<WS>(mask, a[k], p);
        const T rpv = wbcast<WS>(mask, rk, p);
        if constexpr (PIVOT) ok = ok && (pv != T(0)) && isfinite(pv);
        else ok = ok && (pv > T(0)) && isfinite(pv);
        const bool isp = (lane == p);
        const T f = isp ? T(0) : a[k] * rpv;
        if (isp) { used = true; piv_row = k; mypiv = pv; }
#pragma unroll
        for (int j = k + 1; j < NR; ++j) a[j] = fma(-f, wbcast<WS>(mask, a[j], p), a[j]);
        if constexpr (NRHS % 2 == 0) {
#pragma unroll
            for (int j = 0; j < NRHS; j += 2) {
                const T p0 = wbcast<WS>(mask, rhs[j], p), p1 = wbcast<WS>(mask, rhs[j + 1], p);
                ffma2(-f, -f, p0, p1, rhs[j], rhs[j + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < NRHS; ++j) rhs[j] = fma(-f, wbcast<WS>(mask, rhs[j], p), rhs[j]);
        }
    }
    {
        const T inv = rcp_rn(mypiv);
#pragma unroll
        for (int j = 0; j < NRHS; ++j) rhs[j] *= inv;
    }
    if constexpr (!PIVOT) piv_row = lane < nrows ? lane : -1;
    if constexpr (FULLWARP) {
        // uniform within the worker: AND over its WS lanes
        unsigned v = ok ? 1u : 0u;
#pragma unroll
        for (int off = WS / 2; off >= 1; off >>= 1) v &= __shfl_xor_sync(0xffffffffu, v, off, WS);
        return v != 0u;
    } else {
        return __all_sync(mask, ok);
    }
}

// Compact Gauss-Jordan for fully converged warps (mask = all lanes, several WS-lane workers per
// warp): same arithmetic as gauss_jordan<..., FULLWARP = true> but the pivot loop is not unrolled
// (column k of the lane's row is extracted with selects and every column is updated, the pivot
// row's already-eliminated columns being zero), so the code is ~NR times smaller and the loop body
// stays resident in the instruction cache.
template <typename T, int WS, int NR, int NRHS, bool PIVOT>
__device__ __forceinline__ bool gauss_jordan_compact(T (&a)[NR], T (&rhs)[NRHS], int lane, int &piv_row) {
    bool used = lane >= NR;
    bool ok = true;
    piv_row = -1;
    T mypiv = T(1);
#pragma unroll 1
    for (int k = 0; k < NR; ++k) {
        T ak = a[0];
#pragma unroll
        for (int j = 1; j < NR; ++j) ak = (j == k) ? a[j] : ak;
        int p;
        if constexpr (PIVOT) {
            const unsigned key = used ? 0u : ((__float_as_uint(fabsf((float)ak)) & 0xFFFFFFE0u) | (31u - (unsigned)lane));
            unsigned best = key;
#pragma unroll
            for (int off = WS / 2; off >= 1; off >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, off, WS));
            p = 31 - (int)(best & 31u);
        } else {
            p = k;
        }
        const T pv = __shfl_sync(0xffffffffu, ak, p, WS);
        if constexpr (PIVOT) ok = ok && (pv != T(0)) && isfinite(pv);
        else ok = ok && (pv > T(0)) && isfinite(pv);
        const bool isp = (lane == p);
        const T f = isp ? T(0) : ak * rcp_rn(pv);
        if (isp) { used = true; piv_row = k; mypiv = pv; }
        if constexpr (NR % 2 == 0) {
#pragma unroll
            for (int j = 0; j < NR; j += 2) {
                const T p0 = __shfl_sync(0xffffffffu, a[j], p, WS), p1 = __shfl_sync(0xffffffffu, a[j + 1], p, WS);
                ffma2(-f, -f, p0, p1, a[j], a[j + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < NR; ++j) a[j] = fma(-f, __shfl_sync(0xffffffffu, a[j], p, WS), a[j]);
        }
        if constexpr (NRHS % 2 == 0) {
#pragma unroll
            for (int j = 0; j < NRHS; j += 2) {
                const T p0 = __shfl_sync(0xffffffffu, rhs[j], p, WS), p1 = __shfl_sync(0xffffffffu, rhs[j + 1], p, WS);
                ffma2(-f, -f, p0, p1, rhs[j], rhs[j + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < NRHS; ++j) rhs[j] = fma(-f, __shfl_sync(0xffffffffu, rhs[j], p, WS), rhs[j]);
        }
    }
    const T inv = rcp_rn(mypiv);
#pragma unroll
    for (int j = 0; j < NRHS; ++j) rhs[j] *= inv;
    if constexpr (!PIVOT) piv_row = lane < NR ? lane : -1;
    unsigned v = ok ? 1u : 0u;
#pragma unroll
    for (int off = WS / 2; off >= 1; off >>= 1) v &= __shfl_xor_sync(0xffffffffu, v, off, WS);
    return v != 0u;
}

// cp.async (LDGSTS) helpers: 16-byte global -> shared copies that complete asynchronously.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPENDING>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPENDING)); }

// Two independent eliminations interleaved step by step (full-warp workers of WS = 16 lanes):
// problem 1 is SPD (no pivoting), problem 2 uses partial pivoting.  Same arithmetic as two calls of
// gauss_jordan<..., FULLWARP = true>, but the dependent chains of the two systems overlap (ILP).
template <typename T, int NR, int NRHS1, int NRHS2>
__device__ __forceinline__ void gauss_jordan_dual(T (&a1)[NR], T (&r1)[NRHS1], T (&a2)[NR], T (&r2)[NRHS2], int lane,
                                                  int &piv1, int &piv2, bool &ok1, bool &ok2) {
    constexpr int WS = 16;
    const unsigned full = 0xffffffffu;
    bool used2 = lane >= NR;
    ok1 = true; ok2 = true;
    piv2 = -1;
    T mp1 = T(1), mp2 = T(1);
    const bool lo = (threadIdx.x & 16) == 0;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const unsigned key = used2 ? 0u : ((__float_as_uint(fabsf((float)a2[k])) & 0xFFFFFFE0u) | (31u - (unsigned)lane));
        const unsigned b0 = __reduce_max_sync(full, lo ? key : 0u);
        const unsigned b1 = __reduce_max_sync(full, lo ? 0u : key);
        const int p2 = 31 - (int)((lo ? b0 : b1) & 31u);
        const int p1 = k;
        const T rk1 = rcp_rn(a1[k]), rk2 = rcp_rn(a2[k]);
        const T pv1 = __shfl_sync(full, a1[k], p1, WS), rp1 = __shfl_sync(full, rk1, p1, WS);
        const T pv2 = __shfl_sync(full, a2[k], p2, WS), rp2 = __shfl_sync(full, rk2, p2, WS);
        ok1 = ok1 && (pv1 > T(0)) && isfinite(pv1);
        ok2 = ok2 && (pv2 != T(0)) && isfinite(pv2);
        const bool isp1 = lane == p1, isp2 = lane == p2;
        const T f1 = isp1 ? T(0) : a1[k] * rp1;
        const T f2 = isp2 ? T(0) : a2[k] * rp2;
        if (isp1) mp1 = pv1;
        if (isp2) { used2 = true; piv2 = k; mp2 = pv2; }
#pragma unroll
        for (int j = k + 1; j < NR; ++j) {
            a1[j] = fma(-f1, __shfl_sync(full, a1[j], p1, WS), a1[j]);
            a2[j] = fma(-f2, __shfl_sync(full, a2[j], p2, WS), a2[j]);
        }
#pragma unroll
        for (int j = 0; j + 1 < NRHS1; j += 2) {
            const T q0 = __shfl_sync(full, r1[j], p1, WS), q1 = __shfl_sync(full, r1[j + 1], p1, WS);
            ffma2(-f1, -f1, q0, q1, r1[j], r1[j + 1]);
        }
        if constexpr (NRHS1 % 2) r1[NRHS1 - 1] = fma(-f1, __shfl_sync(full, r1[NRHS1 - 1], p1, WS), r1[NRHS1 - 1]);
#pragma unroll
        for (int j = 0; j + 1 < NRHS2; j += 2) {
            const T q0 = __shfl_sync(full, r2[j], p2, WS), q1 = __shfl_sync(full, r2[j + 1], p2, WS);
            ffma2(-f2, -f2, q0, q1, r2[j], r2[j + 1]);
        }
        if constexpr (NRHS2 % 2) r2[NRHS2 - 1] = fma(-f2, __shfl_sync(full, r2[NRHS2 - 1], p2, WS), r2[NRHS2 - 1]);
    }
    const T i1 = rcp_rn(mp1), i2 = rcp_rn(mp2);
#pragma unroll
    for (int j = 0; j < NRHS1; ++j) r1[j] *= i1;
#pragma unroll
    for (int j = 0; j < NRHS2; ++j) r2[j] *= i2;
    piv1 = lane < NR ? lane : -1;
    unsigned v = (ok1 ? 1u : 0u) | (ok2 ? 2u : 0u);
#pragma unroll
    for (int off = WS / 2; off >= 1; off >>= 1) v &= __shfl_xor_sync(full, v, off, WS);
    ok1 = (v & 1u) != 0u;
    ok2 = (v & 2u) != 0u;
}

}  // namespace pdilqr
