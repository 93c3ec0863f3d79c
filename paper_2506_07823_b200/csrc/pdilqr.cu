// pdilqr.cu -- host side of libpdilqr.so: the C ABI of include/pdilqr.h.
// Validation, workspace carve-up, kernel dispatch and launch sequencing.  No allocation, no host
// synchronisation in linearize / solve_lq / step (CUDA-graph capturable).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "pdilqr.h"
#include "lq.cuh"
#include "srbd.cuh"
#include "srbd_fused.cuh"
#include "big.cuh"
#include "big_ric.cuh"
#include "adjoint.cuh"
#include "multi.cuh"
#include "segment.cuh"

using namespace pdilqr;

// Build partition: paper_2506_07823_b200/build.py compiles this file once per part, in parallel
// (the kernels of one part do not depend on those of another):
//   0 everything in one translation unit        1 host: C ABI, validation, workspace layout
//   2 f32 kernels for n, m <= 16                3 f64 kernels for n, m <= 16
//   4 f32 large-n kernels (16 < n, m <= 256)    5 f64 large-n kernels
#ifndef PDILQR_PART
#define PDILQR_PART 0
#endif
#define PDILQR_HOST (PDILQR_PART == 0 || PDILQR_PART == 1)
#define PDILQR_SMALL(f64) (PDILQR_PART == 0 || PDILQR_PART == 2 + (f64))
#define PDILQR_BIG(f64) (PDILQR_PART == 0 || PDILQR_PART == 4 + (f64))

namespace pdq {
extern thread_local std::string g_err;  // pdilqr_last_error (defined in the host part)
}

namespace {

using pdq::g_err;

pdilqr_status fail(pdilqr_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
pdilqr_status fail(pdilqr_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

constexpr size_t kAlign = 256;
constexpr int kMaxAlpha = 15;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Kernel instantiation chosen for (n, m): exact 12x12 (SRBD) or a zero-padded bound.
enum Variant { V12 = 0, V4 = 1, V8 = 2, V16 = 3, VBIG = 4 };
constexpr int kBigMax = 256;   // largest n, m of the CTA-level path

bool pick_variant(int n, int m, Variant &v, int &NX, int &NU) {
    if (n == 12 && m == 12) { v = V12; NX = NU = 12; return true; }
    const int d = std::max(n, m);
    if (d <= 4) { v = V4; NX = NU = 4; return true; }
    if (d <= 8) { v = V8; NX = NU = 8; return true; }
    if (d <= 16) { v = V16; NX = NU = 16; return true; }
    if (d <= kBigMax) { v = VBIG; NX = ld_of(n); NU = ld_of(m); return true; }
    return false;
}

struct Layout {
    size_t elems, vslots, Pp, Kk, tel, tslots, dxw, fail, nonfin, pre, info_tmp, stats;
    size_t elems2 = 0;  // large path with leaf_chunk = 1: second element buffer of the tree scan
    size_t kinds_b, kinds_f, ls_part, ls_cnt;  // grid-scan slot kinds, multi-block line-search scratch
    size_t conv, active;                       // pdilqr_solve per-instance state, active counter
    size_t rho;                                // pdilqr_solve Levenberg-Marquardt shift per instance (double)
    size_t qp[11];  // SRBD internal QP buffers (A, Bm, c, Q, R, S, q, r, Pt, pt, dx0)
    size_t dir[3];  // internal direction (dx, du, dlam)
    size_t adj[8];  // adjoint solve: linear terms (q, r, c, pt, dx0) and solution (wx, wu, wl)
    size_t total;
};

}  // namespace

struct ProfRec {
    const char *name;
    cudaEvent_t start, stop;
};

struct pdilqr_ctx {
    pdilqr_config cfg;
    int device;
    Variant var;
    int NX, NU, esz;
    int chunk, Jb, Pv, Jf, Pf;
    char *ws;
    size_t ws_bytes;
    Layout lay;
    SrbdConst K;
    int launches;
    int occ_fold = 4, occ_ls = 4;  // minimum resident CTAs per SM requested from ptxas (register cap: 128)
    int fold_tpb = 64;             // k_srbd_bwd_fold block size (32 / 64 / 128)
    int fused = 1;                 // 1: 2-kernel fused fold path (default), 0: 4-kernel split path
    int linrec = 1;                // fused path: 1 stage-parallel linearisation records + record-fed fold (default),
                                   // 0 linearisation inside the sequential fold (round-1/2 kernel)
    int fold_mode = 2;             // record-fed fold: 2 = two rows per lane / five instances per warp (default),
                                   // 1 = one instance per warp (column halves), 0 = two instances per warp (row per lane)
    int fold_w = 14;               // fold_mode 1: MINB blocks/SM (12/14/16)
    int fold_nw = 4;               // fold_mode 2: instances per warp (2..5)
    int fold_cp = 1;               // fold_mode 2: stance-compacted policy solve (PDILQR_FOLD_CP=0: all 12 pivots)
    int elem_r2 = 0;               // generic LQ, exact 12x12: PDILQR_ELEM_R2=1 -> k_elem_init_r2 (two rows per lane; measured slower)
    int lin_staged = 2;            // k_srbd_lin_rec: 2 = two warps (state / control halves) per 32 stages (default),
                                   // 1 = one thread per stage, records staged in shared memory, 0 = direct 16-byte stores
    int ric_cs = 1;                // large path: CTAs per instance (thread-block cluster size) of k_big_ric
    bool big_legacy = false;       // large path: PDILQR_BIG_LEGACY=1 forces the element/fold/policy kernels
    bool fault_combine = false;    // PDILQR_FAULT_COMBINE=1: negative control of the parity tests
    bool nvtx = false;             // PDILQR_NVTX=1: an NVTX range around every kernel launch (tracing)
    bool big_mma = false;          // large path, f32: warp-level mma.sync 3xTF32 products in k_big_ric (PDILQR_BIG_MMA)
    bool big_tc = false;           // large path, f32: tcgen05 3xTF32 products in k_big_ric (PDILQR_BIG_TC=1);
                                   // off by default: measured slower than the SIMT tiles (K7)
    bool grid_scan = false;        // latency regime: cooperative grid-wide scans + multi-block line search
    int coop_bwd = 0, coop_fwd = 0;  // max co-resident CTAs of the grid scan kernels
    int coop_ks = 0, coop_fks = 0; // ... of the depth-optimal (Kogge-Stone) reverse / forward scans
    bool ks_bwd = false;           // latency regime: Kogge-Stone instead of the Blelloch tree (D9)
    bool ks_split = true;          // ... with one warp per combine (half-warp split of the full rule)
    int coop_ks2 = 0;
    // pdilqr_solve in progress: convergence bookkeeping handed to the update kernels
    int32_t *sc_conv = nullptr, *sc_active = nullptr;
    double *sc_rho = nullptr;
    double sc_tol = 0.0;
    int sc_iter = 0;
    // per-kernel CUDA-event timing (host bookkeeping only; off unless pdilqr_profile(h, 1))
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<ProfRec> recs;
    cudaEvent_t ev_get() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
};

namespace {
// Scoped timing of one kernel launch on `st` when profiling is enabled.
struct Prof {
    pdilqr_ctx *h;
    cudaStream_t st;
    cudaEvent_t e1 = nullptr;
    const char *name;
    Prof(pdilqr_ctx *h_, const char *nm, cudaStream_t s) : h(h_), st(s), name(nm) {
        if (h->nvtx) nvtxRangePushA(name);  // per-phase ranges for external timeline tools
        if (h->prof) {
            e1 = h->ev_get();
            cudaEventRecord(e1, st);
        }
    }
    ~Prof() {
        if (h->prof) {
            cudaEvent_t e2 = h->ev_get();
            cudaEventRecord(e2, st);
            h->recs.push_back(ProfRec{name, e1, e2});
        }
        if (h->nvtx) nvtxRangePop();
    }
};
}  // namespace

namespace {

pdilqr_status check_cfg(const pdilqr_config *c, Variant &v, int &NX, int &NU) {
    if (!c) return fail(PDILQR_ERR_INVALID_ARG, "cfg is NULL");
    if (c->N < 0 || c->batch < 1 || c->n < 1 || c->m < 1)
        return fail(PDILQR_ERR_DIM, "invalid dimensions N=%d n=%d m=%d batch=%d", c->N, c->n, c->m, c->batch);
    if (c->dtype != PDILQR_F32 && c->dtype != PDILQR_F64) return fail(PDILQR_ERR_INVALID_ARG, "unknown dtype %d", (int)c->dtype);
    if (c->model != PDILQR_MODEL_LQ && c->model != PDILQR_MODEL_SRBD && c->model != PDILQR_MODEL_MULTI_SRBD)
        return fail(PDILQR_ERR_INVALID_ARG, "unknown model %d", (int)c->model);
    if (c->model == PDILQR_MODEL_SRBD && (c->n != 12 || c->m != 12))
        return fail(PDILQR_ERR_DIM, "SRBD model needs n = m = 12 (got %d, %d)", c->n, c->m);
    if (c->model == PDILQR_MODEL_MULTI_SRBD) {
        const auto &mp = c->multi;
        if (mp.n_robots < 1 || mp.n_robots > MULTI_MAX_R || c->n != 12 * mp.n_robots || c->m != 12 * mp.n_robots)
            return fail(PDILQR_ERR_DIM, "multi-robot model needs 1 <= n_robots <= %d and n = m = 12 n_robots (got R=%d, n=%d, m=%d)",
                        MULTI_MAX_R, mp.n_robots, c->n, c->m);
        if (!(mp.d_min > 0) || !(mp.weight >= 0) || !(mp.sharpness > 0))
            return fail(PDILQR_ERR_INVALID_ARG, "invalid collision parameters (d_min > 0, weight >= 0, sharpness > 0)");
    }
    if (c->n_alpha < 0 || c->n_alpha > kMaxAlpha) return fail(PDILQR_ERR_INVALID_ARG, "n_alpha must be in [0, %d]", kMaxAlpha);
    if (c->leaf_chunk < 0) return fail(PDILQR_ERR_INVALID_ARG, "leaf_chunk must be >= 0");
    if (!pick_variant(c->n, c->m, v, NX, NU))
        return fail(PDILQR_ERR_UNSUPPORTED, "n = %d, m = %d: dimensions above %d are not supported", c->n, c->m, kBigMax);
    if (v == VBIG && c->model == PDILQR_MODEL_SRBD)
        return fail(PDILQR_ERR_UNSUPPORTED, "the large-dimension path serves LQ and multi-robot handles");
    if (c->model != PDILQR_MODEL_LQ) {
        const auto &s = c->srbd;
        if (!(s.dt >= 0) || !(s.mass > 0) || !(s.barrier_mu > 0) || !(s.barrier_delta > 0))
            return fail(PDILQR_ERR_INVALID_ARG, "invalid SRBD parameters (dt >= 0, mass > 0, barrier mu, delta > 0)");
    }
    return PDILQR_OK;
}

int default_chunk(const pdilqr_config *c) {
    if (c->leaf_chunk > 0) return c->leaf_chunk;
    // Batch-parallelism already fills 148 SMs for large B: fold each instance in one chunk.
    // For small B use the full tree (span 2 ceil(log2 L)).  See DESIGN.md "Scan schedule".
    if (c->batch >= 148) return c->N + 2;
    if (c->model != PDILQR_MODEL_SRBD) return 1;
    // SRBD step, measured crossover (profiles/r2_crossover_b.txt): the fused fold's latency is
    // ~4 us per stage whatever the batch, the tree's time grows with B * L; mid batches take the
    // fold for short horizons and 8-stage chunks for long ones
    const long L = (long)c->N + 2;
    if ((long)c->batch * L <= 2500) return 1;
    return L <= 64 ? c->N + 2 : 8;
}

size_t big_slot(int n, int m) {
    const size_t init = (size_t)m * ld_of(m + 2 * n + 1);
    const size_t fold = (size_t)n * ld_of(n) * 2 + (size_t)n * ld_of(2 * n) + 2 * ld_of(n);
    const size_t pol = (size_t)n * ld_of(m) + (size_t)m * ld_of(m + n + 1) + ld_of(n);
    const size_t ks = (size_t)n * ld_of(3 * n + 1) + (size_t)n * ld_of(n) + 2 * ld_of(n);  // k_bigks_level
    return (std::max({init, fold, pol, ks, ric_slot(n, m)}) + 63) / 64 * 64;
}
constexpr int kBigPersistent = 148 * 4;  // CTAs of the persistent (stage-parallel) big kernels
constexpr size_t kRicSmemMax = 200 * 1024;  // k_big_ric keeps the m x m Cholesky factor in shared memory

Layout make_big_layout(const pdilqr_config *c, int esz) {
    const size_t B = c->batch, N = c->N, n = c->n, m = c->m, LD = ld_of((int)n), LDU = ld_of((int)m);
    Layout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
    L.elems = take(B * (N + 2) * (3 * n * LD + 2 * LD) * esz);
    if (c->leaf_chunk == 1) L.elems2 = take(B * (N + 2) * (3 * n * LD + 2 * LD) * esz);   // tree scan
    L.Pp = take(B * (N + 2) * (n * LD + LD) * esz);
    L.Kk = take(B * (N + 1) * (m * LD + LDU) * esz);
    L.tel = take(B * (N + 1) * (n * LD + LD) * esz);
    L.dxw = take(B * (N + 2) * LD * esz);
    L.vslots = take(std::max((size_t)kBigPersistent, B) * big_slot((int)n, (int)m) * esz);  // scratch slots
    L.fail = take(B * 4);
    L.nonfin = take(B * 4);
    L.pre = take(B * 4);
    L.info_tmp = take(B * 4);
    L.stats = take(B * (3 * (size_t)esz + 8));
    if (c->model == PDILQR_MODEL_MULTI_SRBD) {  // internal QP and direction of the multi-robot step
        const size_t sz[11] = {(N + 1) * n * n, (N + 1) * n * m, (N + 1) * n, (N + 1) * n * n, (N + 1) * m * m,
                               (N + 1) * m * n, (N + 1) * n, (N + 1) * m, n * n, n, n};
        for (int k = 0; k < 11; ++k) L.qp[k] = take(B * sz[k] * esz);
        L.dir[0] = take(B * (N + 2) * n * esz);
        L.dir[1] = take(B * (N + 1) * m * esz);
        L.dir[2] = take(B * (N + 2) * n * esz);
    }
    {  // pdilqr_solve_lq_adjoint: adjoint linear terms and solution, user (unpadded) layouts
        const size_t nB = c->batch, nN = c->N, nn_ = c->n, mm_ = c->m;
        const size_t sz[8] = {(nN + 1) * nn_, (nN + 1) * mm_, (nN + 1) * nn_, nn_, nn_, (nN + 2) * nn_, (nN + 1) * mm_,
                              (nN + 2) * nn_};
        for (int k = 0; k < 8; ++k) L.adj[k] = take(nB * sz[k] * esz);
    }
    L.total = off;
    return L;
}

Layout make_layout(const pdilqr_config *c, int NX, int NU, int esz, int chunk, int &Jb, int &Pv, int &Jf, int &Pf) {
    const size_t B = c->batch, N = c->N;
    if (NX > 16 || NU > 16 || c->n > 16 || c->m > 16) {  // large path: single chunk
        Jb = Jf = 1; Pv = Pf = 1;
        return make_big_layout(c, esz);
    }
    const size_t VEs = 3 * NX * NX + 2 * NX, TEs = NX * NX + NX, KEs = NU * NX + NU;
    Jb = (int)((N + 2 + chunk - 1) / chunk);
    Jf = (int)((N + 1 + chunk - 1) / chunk);
    Pv = Jb > 1 ? pow2ceil(Jb) : 1;
    Pf = Jf > 1 ? pow2ceil(Jf) : 1;
    Layout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
    L.elems = take(B * (N + 2) * VEs * esz);
    L.vslots = take(B * (Jb > 1 ? Pv : 0) * VEs * esz);
    L.Pp = take(B * (N + 2) * TEs * esz);
    L.Kk = take(B * (N + 1) * KEs * esz);
    L.tel = take(B * (N + 1) * TEs * esz);
    L.tslots = take(B * (Jf > 1 ? Pf : 0) * TEs * esz);
    L.dxw = take(B * (N + 2) * NX * esz);
    L.fail = take(B * 4);
    L.nonfin = take(B * 4);
    L.pre = take(B * 4);
    L.info_tmp = take(B * 4);
    L.stats = take(B * (3 * (size_t)esz + 8));
    L.kinds_b = take(B * (size_t)Pv * 4);
    L.kinds_f = take(B * (size_t)Pf * 4);
    L.ls_part = take(B * (size_t)((N + 2 + 31) / 32) * 34 * 8 * (B < 148 ? 16 : 1));  // x alpha groups
    L.ls_cnt = take(B * 4);
    L.conv = take(B * 4);
    L.active = take(8);
    L.rho = take(B * 8);
    const size_t n = c->n, m = c->m;
    if (c->model != PDILQR_MODEL_LQ) {
        const size_t sz[11] = {(N + 1) * n * n, (N + 1) * n * m, (N + 1) * n, (N + 1) * n * n, (N + 1) * m * m,
                               (N + 1) * m * n, (N + 1) * n, (N + 1) * m, n * n, n, n};
        for (int k = 0; k < 11; ++k) L.qp[k] = take(B * sz[k] * esz);
        L.dir[0] = take(B * (N + 2) * n * esz);
        L.dir[1] = take(B * (N + 1) * m * esz);
        L.dir[2] = take(B * (N + 2) * n * esz);
    }
    {  // pdilqr_solve_lq_adjoint: adjoint linear terms and solution, user (unpadded) layouts
        const size_t nB = c->batch, nN = c->N, nn_ = c->n, mm_ = c->m;
        const size_t sz[8] = {(nN + 1) * nn_, (nN + 1) * mm_, (nN + 1) * nn_, nn_, nn_, (nN + 2) * nn_, (nN + 1) * mm_,
                              (nN + 2) * nn_};
        for (int k = 0; k < 8; ++k) L.adj[k] = take(nB * sz[k] * esz);
    }
    L.total = off;
    return L;
}

template <typename T>
LqWork<T> work(pdilqr_ctx *h) {
    LqWork<T> w;
    w.elems = reinterpret_cast<T *>(h->ws + h->lay.elems);
    w.vslots = reinterpret_cast<T *>(h->ws + h->lay.vslots);
    w.Pp = reinterpret_cast<T *>(h->ws + h->lay.Pp);
    w.Kk = reinterpret_cast<T *>(h->ws + h->lay.Kk);
    w.tel = reinterpret_cast<T *>(h->ws + h->lay.tel);
    w.tslots = reinterpret_cast<T *>(h->ws + h->lay.tslots);
    w.dxw = reinterpret_cast<T *>(h->ws + h->lay.dxw);
    w.fail = reinterpret_cast<int32_t *>(h->ws + h->lay.fail);
    w.nonfin = reinterpret_cast<int32_t *>(h->ws + h->lay.nonfin);
    return w;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

pdilqr_status cuda_check(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PDILQR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return PDILQR_OK;
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

namespace {
template <typename T>
LqArgs<T> internal_qp(pdilqr_ctx *h) {
    auto p = [&](int k) { return reinterpret_cast<const T *>(h->ws + h->lay.qp[k]); };
    return LqArgs<T>{p(0), p(1), p(2), p(3), p(4), p(5), p(6), p(7), p(8), p(9), p(10)};
}

template <typename T>
SrbdIter<T> iter_of(const pdilqr_iterate *it) {
    return SrbdIter<T>{reinterpret_cast<const T *>(it->x),    reinterpret_cast<const T *>(it->u),
                       reinterpret_cast<const T *>(it->lam),  reinterpret_cast<const T *>(it->x0),
                       reinterpret_cast<const T *>(it->x_ref), reinterpret_cast<const T *>(it->u_ref),
                       it->contact,                           reinterpret_cast<const T *>(it->feet)};
}

template <typename T>
SrbdIter<T> iter_of(const pdilqr_iterate *it, const pdilqr_ctx *h) {
    SrbdIter<T> r = iter_of<T>(it);
    r.conv = h->sc_conv;
    r.active = h->sc_active;
    r.rho = h->sc_rho;
    r.tol = h->sc_tol;
    r.iter = h->sc_iter;
    return r;
}

}  // namespace

// Entry points of the kernel parts, called from the host part (explicit instantiations below).
namespace pdq {
template <typename T>
pdilqr_status run_big(pdilqr_ctx *h, const LqArgs<T> &qp, LqOut<T> out, int32_t *info, cudaStream_t st);
template <typename T>
pdilqr_status dispatch_lq(pdilqr_ctx *h, const LqArgs<T> &qp, LqOut<T> out, int32_t *info, const int32_t *pre,
                          cudaStream_t st, bool skip_init = false);
template <typename T>
pdilqr_status run_linearize(pdilqr_ctx *h, const pdilqr_iterate *it, const LqArgs<T> &outq, int32_t *pre,
                            cudaStream_t st);
template <typename T>
pdilqr_status run_step(pdilqr_ctx *h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir, cudaStream_t st);
template <typename T>
pdilqr_status run_adjoint(pdilqr_ctx *h, const LqArgs<T> &qp, const LqOut<T> &sol, const T *gdx, const T *gdu,
                          const T *gdl, const AdjGrad<T> &grad, int32_t *info, cudaStream_t st);
// k_big_ric cluster-size probe: true if a cluster of cs CTAs with smem bytes can be co-scheduled
template <typename T>
bool ric_cluster_fits(int cs, size_t smem, bool ut);
cudaError_t debug_tc_gemm(int M, int N, int K, int ta, int tb, const float *A, int lda, const float *Bm, int ldb,
                          const float *Cin, float *C, cudaStream_t st);
// centralized multi-robot model (multi.cuh): linearisation and one SQP step
template <typename T>
pdilqr_status run_multi_linearize(pdilqr_ctx *h, const pdilqr_iterate *it, const LqArgs<T> &outq, int32_t *pre,
                                  cudaStream_t st);
template <typename T>
pdilqr_status run_multi_step(pdilqr_ctx *h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir, cudaStream_t st);
// horizon sharding (segment.cuh), n, m <= 16 handles
template <typename T>
pdilqr_status run_seg_reduce(pdilqr_ctx *h, const LqArgs<T> &qp, T *S_out, int32_t *info, cudaStream_t st);
template <typename T>
pdilqr_status run_seg_suffix(pdilqr_ctx *h, const T *S_all, int G, int r, const T *Pt, const T *pt, T *P_out, T *p_out,
                             cudaStream_t st);
template <typename T>
pdilqr_status run_seg_forward(pdilqr_ctx *h, const LqArgs<T> &qp, T *F_out, cudaStream_t st);
template <typename T>
pdilqr_status run_seg_prefix(pdilqr_ctx *h, const T *F_all, int G, int r, const T *dx0, T *dxs, cudaStream_t st);
// co-resident CTAs of the cooperative latency-regime scan kernels (v: Variant)
template <typename T>
void grid_occupancy(int v, int sms, int &nb, int &nf, int &nk, int &nfk, int &nk2);
}  // namespace pdq

#if PDILQR_SMALL(0) || PDILQR_SMALL(1)
namespace pdq {
// --------------------------------------------------------------------------- LQ pipeline
template <typename T, int NX, int NU, bool EX>
pdilqr_status run_lq(pdilqr_ctx *h, const LqArgs<T> &qp, LqOut<T> out, int32_t *info, const int32_t *pre,
                     cudaStream_t st, bool skip_init) {
    constexpr int WS = worker_width(NX > NU ? NX : NU);
    constexpr int WSX = worker_width(NX);
    const int B = h->cfg.batch, N = h->cfg.N, n = h->cfg.n, m = h->cfg.m;
    LqWork<T> ws = work<T>(h);
    if (!skip_init) cudaMemsetAsync(ws.fail, 0x7f, (size_t)B * 4, st);
    cudaMemsetAsync(ws.nonfin, 0, (size_t)B * 4, st);
    int launches = 0;
    if (!skip_init) {  // element init
        const int wpb = 128 / WS;
        const long nw = (long)B * (N + 2);
        Prof pf(h, "k_elem_init", st);
        bool done = false;
        if constexpr (EX && NX == 12 && NU == 12) {
            if (h->elem_r2 && qp.S) {   // two rows per lane, 8 items per 64-thread block
                const size_t smem2 = 8 * sizeof(ElemR2Smem<T>);
                set_smem(k_elem_init_r2<T>, smem2);
                k_elem_init_r2<T><<<(unsigned)((nw + 7) / 8), 64, smem2, st>>>(qp, B, N, ws);
                done = true;
            }
        }
        if (!done) {
            const size_t smem = (size_t)wpb * elem_init_smw<NX, NU, EX>() * sizeof(T);
            set_smem(k_elem_init<T, NX, NU, EX>, smem);
            k_elem_init<T, NX, NU, EX><<<(unsigned)((nw + wpb - 1) / wpb), wpb * WS, smem, st>>>(qp, B, N, n, m, ws);
        }
        ++launches;
        if (h->fault_combine) {  // negative control (tests only): corrupt one element of instance 0
            k_fault_inject<T, NX><<<1, 1, 0, st>>>(ws, N);
            ++launches;
        }
    }
    bool bwd_done = false;
    if constexpr (WSX == 16) {
        if (h->Jb > 1 && h->grid_scan && h->ks_bwd && h->ks_split) {  // Kogge-Stone, one warp per combine (D9)
            int Pv = h->Pv, Bv = B, Nv = N;
            const size_t smem = 4 * sizeof(CombineSmem<T, NX>);
            set_smem(k_scan_bwd_ks2<T, NX>, smem);
            const long units = (long)B * (N + 2);
            const int grid = (int)std::max(1L, std::min((long)h->coop_ks2, (units + 3) / 4));
            void *args[] = {&Bv, &Nv, &Pv, &ws};
            Prof pf(h, "k_scan_bwd_ks2", st);
            cudaLaunchCooperativeKernel((const void *)k_scan_bwd_ks2<T, NX>, grid, 128, args, smem, st);
            ++launches;
            bwd_done = true;
        }
    }
    if (bwd_done) {
    } else if (h->Jb == 1) {  // single chunk: tight per-instance fold with prefetch
        const size_t smem = (size_t)(128 / WSX) * sizeof(FoldChainSmem<T, NX>);
        set_smem(k_fold<T, NX, 4>, smem);
        Prof pf(h, "k_fold", st);
        const int ipb = 128 / WSX;
        k_fold<T, NX, 4><<<(B + ipb - 1) / ipb, 128, smem, st>>>(B, N, ws);
        ++launches;
    } else if (h->grid_scan && h->ks_bwd) {  // cooperative depth-optimal scan (latency regime, D9)
        int Pv = h->Pv, Bv = B, Nv = N;
        const int wpb = 128 / WSX;
        const size_t smem = wpb * sizeof(CombineSmem<T, NX>);
        set_smem(k_scan_bwd_ks<T, NX>, smem);
        const long units = (long)B * (N + 2);
        const int grid = (int)std::max(1L, std::min((long)h->coop_ks, (units + wpb - 1) / wpb));
        void *args[] = {&Bv, &Nv, &Pv, &ws};
        Prof pf(h, "k_scan_bwd_ks", st);
        cudaLaunchCooperativeKernel((const void *)k_scan_bwd_ks<T, NX>, grid, 128, args, smem, st);
        ++launches;
    } else if (h->grid_scan) {  // cooperative grid-wide tree (latency regime)
        int J = h->Jb, Pv = h->Pv, chunk = h->chunk, Bv = B, Nv = N;
        int *kinds = reinterpret_cast<int *>(h->ws + h->lay.kinds_b);
        const int wpb = 128 / WSX;
        const size_t smem = wpb * sizeof(CombineSmem<T, NX>);
        set_smem(k_scan_bwd_grid<T, NX>, smem);
        const long units = (long)B * std::max(J, Pv / 2);
        const int grid = (int)std::max(1L, std::min((long)h->coop_bwd, (units + wpb - 1) / wpb));
        void *args[] = {&Bv, &Nv, &chunk, &J, &Pv, &ws, &kinds};
        Prof pf(h, "k_scan_bwd_grid", st);
        cudaLaunchCooperativeKernel((const void *)k_scan_bwd_grid<T, NX>, grid, 128, args, smem, st);
        ++launches;
    } else {  // backward scan
        const int J = h->Jb, Pv = h->Pv;
        const size_t cs = sizeof(CombineSmem<T, NX>);
        int W = 1, IPB = 8;
        if (J > 1) {
            W = std::max(J - 1, Pv / 2);
            W = std::min({W, (int)(200 * 1024 / cs), 256 / WSX});
            W = std::max(W, 1);
            IPB = std::max(1, std::min(8, 128 / (W * WSX)));
        }
        const size_t smem = (size_t)IPB * W * cs + (size_t)IPB * Pv * sizeof(int);
        set_smem(k_scan_bwd<T, NX>, smem);
        Prof pf(h, "k_scan_bwd", st);
        k_scan_bwd<T, NX><<<(B + IPB - 1) / IPB, IPB * W * WSX, smem, st>>>(B, N, h->chunk, J, Pv, W, IPB, ws);
        ++launches;
    }
    {  // policy
        const int wpb = 128 / WS;
        const long nw = (long)B * (N + 1);
        const size_t smem = (size_t)wpb * (NX * NU + NX * NX + NX * NU + NU * NX + round_up4(NU) + NX + NX) * sizeof(T);
        set_smem(k_policy<T, NX, NU, EX>, smem);
        Prof pf(h, "k_policy", st);
        k_policy<T, NX, NU, EX><<<(unsigned)((nw + wpb - 1) / wpb), wpb * WS, smem, st>>>(qp, B, N, n, m, ws, out);
        ++launches;
    }
    if (h->grid_scan && h->ks_bwd && h->Jf > 1) {  // cooperative depth-optimal forward scan (D9)
        int Pf = h->Pf, Bv = B, Nv = N, nv = n;
        const int wpb = 128 / WSX;
        const size_t smem = wpb * sizeof(FwdSmem<T, NX>);
        set_smem(k_scan_fwd_ks<T, NX>, smem);
        const long units = (long)B * (N + 1);
        const int grid = (int)std::max(1L, std::min((long)h->coop_fks, (units + wpb - 1) / wpb));
        const T *dx0 = qp.dx0;
        T *dxo = out.dx;
        void *args[] = {&dx0, &Bv, &Nv, &nv, &Pf, &ws, &dxo};
        Prof pf(h, "k_scan_fwd_ks", st);
        cudaLaunchCooperativeKernel((const void *)k_scan_fwd_ks<T, NX>, grid, 128, args, smem, st);
        ++launches;
    } else if (h->grid_scan && h->Jf > 1) {  // cooperative grid-wide forward tree
        int J = h->Jf, Pf = h->Pf, chunk = h->chunk, Bv = B, Nv = N, nv = n;
        int *kinds = reinterpret_cast<int *>(h->ws + h->lay.kinds_f);
        const int wpb = 128 / WSX;
        const size_t smem = wpb * sizeof(FwdSmem<T, NX>);
        set_smem(k_scan_fwd_grid<T, NX>, smem);
        const long units = (long)B * std::max(J, Pf / 2);
        const int grid = (int)std::max(1L, std::min((long)h->coop_fwd, (units + wpb - 1) / wpb));
        const T *dx0 = qp.dx0;
        T *dxo = out.dx;
        void *args[] = {&dx0, &Bv, &Nv, &nv, &chunk, &J, &Pf, &ws, &dxo, &kinds};
        Prof pf(h, "k_scan_fwd_grid", st);
        cudaLaunchCooperativeKernel((const void *)k_scan_fwd_grid<T, NX>, grid, 128, args, smem, st);
        ++launches;
    } else {  // forward scan
        const int J = h->Jf, Pf = h->Pf;
        const size_t cs = sizeof(FwdSmem<T, NX>);
        int W = 1, IPB = 8;
        if (J > 1) {
            W = std::max(J, Pf / 2);
            W = std::min({W, (int)(200 * 1024 / cs), 256 / WSX});
            W = std::max(W, 1);
            IPB = std::max(1, std::min(8, 128 / (W * WSX)));
        }
        const size_t smem = (size_t)IPB * W * cs + (size_t)IPB * Pf * sizeof(int);
        set_smem(k_scan_fwd<T, NX>, smem);
        Prof pf(h, "k_scan_fwd", st);
        k_scan_fwd<T, NX><<<(B + IPB - 1) / IPB, IPB * W * WSX, smem, st>>>(qp.dx0, B, N, n, h->chunk, J, Pf, W, IPB, ws,
                                                                            out.dx);
        ++launches;
    }
    {  // du, dlam
        const long tot = (long)B * ((long)(N + 1) * m + (long)(N + 2) * n);
        Prof pf(h, "k_tail", st);
        k_tail<T, NX, NU><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(B, N, n, m, ws, out);
        ++launches;
    }
    if (info) {
        Prof pf(h, "k_finalize_info", st);
        k_finalize_info<<<(B + 255) / 256, 256, 0, st>>>(B, ws.fail, ws.nonfin, pre, info);
        ++launches;
    }
    h->launches += launches;
    return cuda_check("solve_lq launch");
}

// Large dimensions (16 < max(n, m) <= 256): CTA-level single-chunk path (big.cuh).
template <typename T>
pdilqr_status dispatch_lq(pdilqr_ctx *h, const LqArgs<T> &qp, LqOut<T> out, int32_t *info, const int32_t *pre,
                          cudaStream_t st, bool skip_init) {
    switch (h->var) {
        case V12: return run_lq<T, 12, 12, true>(h, qp, out, info, pre, st, skip_init);
        case V4: return run_lq<T, 4, 4, false>(h, qp, out, info, pre, st, skip_init);
        case V8: return run_lq<T, 8, 8, false>(h, qp, out, info, pre, st, skip_init);
        case V16: return run_lq<T, 16, 16, false>(h, qp, out, info, pre, st, skip_init);
        default: return run_big<T>(h, qp, out, info, st);
    }
}

template <typename T>
pdilqr_status run_linearize(pdilqr_ctx *h, const pdilqr_iterate *it, const LqArgs<T> &outq, int32_t *pre,
                            cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N;
    cudaMemsetAsync(pre, 0, (size_t)B * 4, st);
    const long nw = (long)B * (N + 2);
    {
    Prof pf(h, "k_srbd_linearize", st);
    k_srbd_linearize<T><<<(unsigned)((nw + 7) / 8), 128, 0, st>>>(h->K, iter_of<T>(it), B, N, outq, pre);
    }
    h->launches += 1;
    return cuda_check("linearize launch");
}

// Single-chunk schedule, split path (4 kernels): stage-parallel linearisation + element init,
// per-instance fold, stage-parallel policy, per-instance rollout + line search + update.
template <typename T>
pdilqr_status run_step_split(pdilqr_ctx *h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir,
                             cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N;
    LqWork<T> ws = work<T>(h);
    int32_t *pre = reinterpret_cast<int32_t *>(h->ws + h->lay.pre);
    LqArgs<T> qp = internal_qp<T>(h);
    qp.S = nullptr;
    T *dx, *du, *dl;
    if (dir && dir->dx) {
        dx = (T *)dir->dx; du = (T *)dir->du; dl = (T *)dir->dlam;
    } else {
        dx = reinterpret_cast<T *>(h->ws + h->lay.dir[0]);
        du = reinterpret_cast<T *>(h->ws + h->lay.dir[1]);
        dl = reinterpret_cast<T *>(h->ws + h->lay.dir[2]);
    }
    cudaMemsetAsync(ws.fail, 0x7f, (size_t)B * 4, st);
    cudaMemsetAsync(pre, 0, (size_t)B * 4, st);
    {
        const long nw = (long)B * (N + 2);
        const size_t smem = 8 * sizeof(LinElemSmem<T>);
        set_smem(k_srbd_lin_elem<T>, smem);
        Prof pf(h, "k_srbd_lin_elem", st);
        k_srbd_lin_elem<T><<<(unsigned)((nw + 7) / 8), 128, smem, st>>>(h->K, iter_of<T>(it, h), B, N, ws, qp, pre);
    }
    {
        const size_t smem = 8 * sizeof(FoldChainSmem<T, 12>);
        set_smem(k_fold<T, 12, 4>, smem);
        Prof pf(h, "k_fold", st);
        k_fold<T, 12, 4><<<(B + 7) / 8, 128, smem, st>>>(B, N, ws);
    }
    {
        LqOut<T> out{dx, du, dl, dir ? (T *)dir->K : nullptr, dir ? (T *)dir->k : nullptr};
        const size_t smem = (size_t)8 * (12 * 12 * 4 + 12 + 12 + 12) * sizeof(T);
        set_smem(k_policy<T, 12, 12, true>, smem);
        Prof pf(h, "k_policy", st);
        const long nw = (long)B * (N + 1);
        k_policy<T, 12, 12, true><<<(unsigned)((nw + 7) / 8), 128, smem, st>>>(qp, B, N, 12, 12, ws, out);
    }
    {
        LsOut<T> so{(T *)stats->cost, (T *)stats->theta, (T *)stats->alpha, stats->accepted, stats->info};
        Prof pf(h, "k_srbd_fwd_ls", st);
        constexpr int WPB = LsWarps<T>::value;
        k_srbd_fwd_ls<T, 4><<<(B + WPB - 1) / WPB, 32 * WPB, 0, st>>>(h->K, iter_of<T>(it, h), B, N, ws, dx, du, dl, nullptr, so,
                                                                       pre);
    }
    h->launches += 4;
    return cuda_check("step (split) launch");
}

// Single-chunk schedule: the fused fold path (srbd_fused.cuh), 2 kernels per step.
template <typename T>
pdilqr_status run_step_fused(pdilqr_ctx *h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir, cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N;
    LqWork<T> ws = work<T>(h);
    int32_t *info_tmp = reinterpret_cast<int32_t *>(h->ws + h->lay.info_tmp);
    T *dx, *du, *dl;
    if (dir && dir->dx) {
        dx = (T *)dir->dx; du = (T *)dir->du; dl = (T *)dir->dlam;
    } else {
        dx = reinterpret_cast<T *>(h->ws + h->lay.dir[0]);
        du = reinterpret_cast<T *>(h->ws + h->lay.dir[1]);
        dl = reinterpret_cast<T *>(h->ws + h->lay.dir[2]);
    }
    if (h->linrec) {
        // stage-parallel linearisation records (ws.elems is free on the single-chunk path)
        T *rec = ws.elems;
        {
            const long tot = (long)B * (N + 1);
            Prof pf(h, "k_srbd_lin_rec", st);
            if (h->lin_staged == 2) {   // two warps per 32 stages (state / control halves)
                const size_t smem = (size_t)32 * (LinRec::SIZE + 16 / sizeof(T)) * sizeof(T);
                set_smem(k_srbd_lin_rec2<T>, smem);
                k_srbd_lin_rec2<T><<<(unsigned)((tot + 31) / 32), 64, smem, st>>>(h->K, iter_of<T>(it, h), B, N, rec);
            } else if (h->lin_staged) {
                constexpr int TPB = 32;
                const size_t smem = (size_t)TPB * (LinRec::SIZE + 16 / sizeof(T)) * sizeof(T);
                set_smem(k_srbd_lin_rec<T, true>, smem);
                k_srbd_lin_rec<T, true><<<(unsigned)((tot + TPB - 1) / TPB), TPB, smem, st>>>(h->K, iter_of<T>(it, h), B, N, rec);
            } else {
                constexpr int TPB = 128;
                k_srbd_lin_rec<T, false><<<(unsigned)((tot + TPB - 1) / TPB), TPB, 0, st>>>(h->K, iter_of<T>(it, h), B, N, rec);
            }
        }
        Prof pf(h, "k_srbd_bwd_fold", st);
        if (h->fold_mode == 2) {   // two rows per lane, five instances per warp (default)
            auto g2 = [&](auto kern, int nw, size_t slice) {
                const size_t smem = (size_t)nw * slice;
                set_smem(kern, smem);
                kern<<<(B + nw - 1) / nw, 32, smem, st>>>(h->K, iter_of<T>(it, h), B, N, ws, rec, info_tmp);
            };
            if (!h->fold_cp) g2(k_srbd_bwd_fold_r2<T, 4, false>, 4, sizeof(FoldR2Smem<T, 4>));
            else switch (h->fold_nw) {
                case 2: g2(k_srbd_bwd_fold_r2<T, 2>, 2, sizeof(FoldR2Smem<T, 2>)); break;
                case 3: g2(k_srbd_bwd_fold_r2<T, 3>, 3, sizeof(FoldR2Smem<T, 3>)); break;
                case 5: g2(k_srbd_bwd_fold_r2<T, 5>, 5, sizeof(FoldR2Smem<T, 5>)); break;
                default: g2(k_srbd_bwd_fold_r2<T, 4>, 4, sizeof(FoldR2Smem<T, 4>)); break;
            }
        } else if (h->fold_mode == 1) {   // one instance per warp (two lanes per row)
            auto gw = [&](auto kern) {
                const size_t smem = 2 * sizeof(FoldWSmem<T>);
                set_smem(kern, smem);
                kern<<<(B + 1) / 2, 64, smem, st>>>(h->K, iter_of<T>(it, h), B, N, ws, rec, info_tmp);
            };
            switch (h->fold_w) {
                case 12: gw(k_srbd_bwd_fold_w<T, 12>); break;
                case 16: gw(k_srbd_bwd_fold_w<T, 16>); break;
                default: gw(k_srbd_bwd_fold_w<T, 14>); break;
            }
        } else {
        auto go = [&](auto kern, int tpb) {
            const int ipb = tpb / 16;
            const size_t smem = (size_t)ipb * sizeof(FoldRecSmem<T>);
            set_smem(kern, smem);
            kern<<<(B + ipb - 1) / ipb, tpb, smem, st>>>(h->K, iter_of<T>(it, h), B, N, ws, rec, info_tmp);
        };
        switch (h->occ_fold * 1000 + h->fold_tpb) {
            case 4064: go(k_srbd_bwd_fold_rec<T, 4, 64>, 64); break;
            case 6064: go(k_srbd_bwd_fold_rec<T, 6, 64>, 64); break;
            default: go(k_srbd_bwd_fold_rec<T, 5, 64>, 64); break;
        }
        }
        h->launches += 1;
    } else {
        Prof pf(h, "k_srbd_bwd_fold", st);
        auto go = [&](auto kern, int tpb) {
            const int ipb = tpb / 16;  // instances per block
            const size_t smem = (size_t)ipb * sizeof(FoldSmem<T>);
            set_smem(kern, smem);
            kern<<<(B + ipb - 1) / ipb, tpb, smem, st>>>(h->K, iter_of<T>(it, h), B, N, ws, info_tmp);
        };
        if (h->sc_rho) go(k_srbd_bwd_fold<T, 4, 64, true>, 64);   // pdilqr_solve: Levenberg-Marquardt ladder
        else switch (h->occ_fold * 1000 + h->fold_tpb) {
            case 4032: go(k_srbd_bwd_fold<T, 4, 32>, 32); break;
            case 4128: go(k_srbd_bwd_fold<T, 4, 128>, 128); break;
            case 3064: go(k_srbd_bwd_fold<T, 3, 64>, 64); break;
            case 2064: go(k_srbd_bwd_fold<T, 2, 64>, 64); break;
            default: go(k_srbd_bwd_fold<T, 4, 64>, 64); break;
        }
    }
    {
        LsOut<T> so{(T *)stats->cost, (T *)stats->theta, (T *)stats->alpha, stats->accepted, stats->info};
        Prof pf(h, "k_srbd_fwd_ls", st);
        auto go = [&](auto kern) {
            constexpr int WPB = LsWarps<T>::value;
            kern<<<(B + WPB - 1) / WPB, 32 * WPB, 0, st>>>(h->K, iter_of<T>(it, h), B, N, ws, dx, du, dl, info_tmp, so, nullptr);
        };
        switch (sizeof(T) == 8 ? 2 : h->occ_ls) {   // fp64: 2 blocks/SM (the 128-register cap spills)
            case 3: go(k_srbd_fwd_ls<T, 3>); break;
            case 4: go(k_srbd_fwd_ls<T, 4>); break;
            case 5: go(k_srbd_fwd_ls<T, 5>); break;
            default: go(k_srbd_fwd_ls<T, 2>); break;
        }
    }
    if (dir && dir->dx && (dir->K || dir->k)) {  // optional policy export (row-major [B][N+1][m][n] / [m])
        const size_t KS = KE<12, 12>::SIZE;
        if (dir->K)
            cudaMemcpy2DAsync(dir->K, 144 * sizeof(T), ws.Kk, KS * sizeof(T), 144 * sizeof(T), (size_t)B * (N + 1),
                              cudaMemcpyDeviceToDevice, st);
        if (dir->k)
            cudaMemcpy2DAsync(dir->k, 12 * sizeof(T), ws.Kk + 144, KS * sizeof(T), 12 * sizeof(T), (size_t)B * (N + 1),
                              cudaMemcpyDeviceToDevice, st);
    }
    h->launches += 2;
    return cuda_check("step (fused) launch");
}

template <typename T>
pdilqr_status run_step(pdilqr_ctx *h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir, cudaStream_t st) {
    if (h->Jb == 1 && h->cfg.n == 12 && h->cfg.m == 12)
        return h->fused ? run_step_fused<T>(h, it, stats, dir, st) : run_step_split<T>(h, it, stats, dir, st);
    const int B = h->cfg.batch, N = h->cfg.N;
    LqArgs<T> qp = internal_qp<T>(h);
    int32_t *pre = reinterpret_cast<int32_t *>(h->ws + h->lay.pre);
    int32_t *info_tmp = reinterpret_cast<int32_t *>(h->ws + h->lay.info_tmp);
    pdilqr_status s = PDILQR_OK;
    if (h->cfg.n == 12 && h->cfg.m == 12) {
        // SRBD: linearisation fused with element init (stage-parallel); the LQ pipeline below
        // then starts at the scan (S = 0 is passed as NULL)
        LqWork<T> ws = work<T>(h);
        cudaMemsetAsync(ws.fail, 0x7f, (size_t)B * 4, st);
        cudaMemsetAsync(pre, 0, (size_t)B * 4, st);
        const long nw = (long)B * (N + 2);
        const size_t smem = 8 * sizeof(LinElemSmem<T>);
        set_smem(k_srbd_lin_elem<T>, smem);
        {
            Prof pf(h, "k_srbd_lin_elem", st);
            k_srbd_lin_elem<T><<<(unsigned)((nw + 7) / 8), 128, smem, st>>>(h->K, iter_of<T>(it, h), B, N, ws, qp, pre);
        }
        h->launches += 1;
        qp.S = nullptr;
    } else {
        s = run_linearize<T>(h, it, qp, pre, st);
        if (s != PDILQR_OK) return s;
    }
    LqOut<T> out;
    if (dir && dir->dx) {
        out = LqOut<T>{(T *)dir->dx, (T *)dir->du, (T *)dir->dlam, (T *)dir->K, (T *)dir->k};
    } else {
        out = LqOut<T>{reinterpret_cast<T *>(h->ws + h->lay.dir[0]), reinterpret_cast<T *>(h->ws + h->lay.dir[1]),
                       reinterpret_cast<T *>(h->ws + h->lay.dir[2]), nullptr, nullptr};
    }
    // latency regime: the line search's last warp derives the info word itself (no k_finalize_info)
    int32_t *lq_info = h->grid_scan ? nullptr : info_tmp;
    s = (h->cfg.n == 12 && h->cfg.m == 12) ? dispatch_lq<T>(h, qp, out, lq_info, pre, st, /*skip_init=*/true)
                                           : dispatch_lq<T>(h, qp, out, lq_info, pre, st);
    if (s != PDILQR_OK) return s;
    LsOut<T> so{(T *)stats->cost, (T *)stats->theta, (T *)stats->alpha, stats->accepted, stats->info};
    if (h->grid_scan) {
        const int S = (N + 2 + 31) / 32;
        // alpha groups: spread the n_alpha + 1 slots over blocks while the grid stays within ~4 warps/SM
        const int AG = B < 148 ? std::max(1, std::min(h->cfg.n_alpha + 1, (148 * 4) / (B * S))) : 1;
        double *part = reinterpret_cast<double *>(h->ws + h->lay.ls_part);
        int *cnt = reinterpret_cast<int *>(h->ws + h->lay.ls_cnt);
        cudaMemsetAsync(cnt, 0, (size_t)B * 4, st);
        Prof pf(h, "k_srbd_ls_multi", st);
        const int32_t *fail = reinterpret_cast<const int32_t *>(h->ws + h->lay.fail);
        const int32_t *nonfin = reinterpret_cast<const int32_t *>(h->ws + h->lay.nonfin);
        k_srbd_ls_multi<T><<<dim3(S * AG, B), 32, 0, st>>>(h->K, iter_of<T>(it, h), B, N, out.dx, out.du, out.dlam, nullptr,
                                                           so, part, cnt, AG, fail, nonfin, pre);
    } else {
        Prof pf(h, "k_srbd_linesearch", st);
        k_srbd_linesearch<T><<<(B + 3) / 4, 128, 0, st>>>(h->K, iter_of<T>(it, h), B, N, out.dx, out.du, out.dlam, info_tmp, so);
    }
    h->launches += 1;
    return cuda_check("step launch");
}


// Adjoint of solve_lq (adjoint.cuh): linear terms from the upstream gradient, the same scans on
// the handle's matrices, then the outer-product gradients.
template <typename T>
pdilqr_status run_adjoint(pdilqr_ctx *h, const LqArgs<T> &qp, const LqOut<T> &sol, const T *gdx, const T *gdu,
                          const T *gdl, const AdjGrad<T> &grad, int32_t *info, cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N, n = h->cfg.n, m = h->cfg.m;
    auto ws = [&](int k) { return reinterpret_cast<T *>(h->ws + h->lay.adj[k]); };
    AdjRhs<T> rhs{ws(0), ws(1), ws(2), ws(3), ws(4)};
    const long tr = (long)B * ((long)(N + 2) * n * 2 + (long)(N + 1) * m);
    {
        Prof pf(h, "k_adj_rhs", st);
        k_adj_rhs<T><<<(unsigned)std::min<long>((tr + 255) / 256, 148L * 16), 256, 0, st>>>(B, N, n, m, gdx, gdu, gdl, rhs);
    }
    h->launches += 1;
    LqArgs<T> aq = qp;
    aq.q = rhs.q; aq.r = rhs.r; aq.c = rhs.c; aq.pt = rhs.pt; aq.dx0 = rhs.dx0;
    LqOut<T> w{ws(5), ws(6), ws(7), nullptr, nullptr};
    pdilqr_status s = dispatch_lq<T>(h, aq, w, info, nullptr, st);
    if (s != PDILQR_OK) return s;
    const long nn = (long)n * n, nm = (long)n * m, mm = (long)m * m;
    const long tg = (long)B * ((long)(N + 1) * (2 * nn + 2 * nm + mm + 2 * n + m) + nn + 2 * n);
    {
        Prof pf(h, "k_adj_grad", st);
        AdjIn<T> z{sol.dx, sol.du, sol.dlam, w.dx, w.du, w.dlam};
        k_adj_grad<T><<<(unsigned)std::min<long>((tg + 255) / 256, 148L * 16), 256, 0, st>>>(B, N, n, m, z, grad);
    }
    h->launches += 1;
    return cuda_check("solve_lq_adjoint launch");
}

// --------------------------------------------------------------------------- horizon sharding
#define PDILQR_SEG_DISPATCH(...)                                             \
    switch (h->var) {                                                        \
        case V12: { constexpr int NX = 12, WS = 16; __VA_ARGS__; } break;    \
        case V4: { constexpr int NX = 4, WS = 4; __VA_ARGS__; } break;       \
        case V8: { constexpr int NX = 8, WS = 8; __VA_ARGS__; } break;       \
        case V16: { constexpr int NX = 16, WS = 16; __VA_ARGS__; } break;    \
        default: return fail(PDILQR_ERR_UNSUPPORTED, "horizon sharding serves n, m <= 16"); \
    }

template <typename T>
pdilqr_status run_seg_reduce(pdilqr_ctx *h, const LqArgs<T> &qp, T *S_out, int32_t *info, cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N, n = h->cfg.n, m = h->cfg.m;
    LqWork<T> ws = work<T>(h);
    cudaMemsetAsync(ws.fail, 0x7f, (size_t)B * 4, st);
    h->launches = 0;
    PDILQR_SEG_DISPATCH({
        constexpr int NU = NX;
        const bool ex = h->var == V12;
        const int wpb = 128 / WS;
        const long nw = (long)B * (N + 2);
        const size_t smem = (size_t)wpb * elem_init_smw<NX, NU, true>() * sizeof(T);
        {
            Prof pf(h, "k_elem_init", st);
            if (ex) {
                set_smem(k_elem_init<T, NX, NU, true>, smem);
                k_elem_init<T, NX, NU, true><<<(unsigned)((nw + wpb - 1) / wpb), wpb * WS, smem, st>>>(qp, B, N, n, m, ws);
            } else {
                set_smem(k_elem_init<T, NX, NU, false>, smem);
                k_elem_init<T, NX, NU, false><<<(unsigned)((nw + wpb - 1) / wpb), wpb * WS, smem, st>>>(qp, B, N, n, m, ws);
            }
        }
        const size_t sm2 = (size_t)(128 / WS) * sizeof(CombineSmem<T, NX>);
        set_smem(k_seg_reduce<T, NX, WS>, sm2);
        {
            Prof pf(h, "k_seg_reduce", st);
            k_seg_reduce<T, NX, WS><<<B, 128, sm2, st>>>(B, N, n, ws, S_out);
        }
    })
    if (info) k_finalize_info<<<(B + 255) / 256, 256, 0, st>>>(B, ws.fail, ws.nonfin, nullptr, info);
    h->launches = info ? 3 : 2;
    return cuda_check("segment reduce launch");
}

template <typename T>
pdilqr_status run_seg_suffix(pdilqr_ctx *h, const T *S_all, int G, int r, const T *Pt, const T *pt, T *P_out, T *p_out,
                             cudaStream_t st) {
    const int B = h->cfg.batch, n = h->cfg.n;
    LqWork<T> ws = work<T>(h);
    PDILQR_SEG_DISPATCH({
        const int wpb = 128 / WS;
        const size_t sm = (size_t)wpb * sizeof(CombineSmem<T, NX>);
        set_smem(k_seg_suffix<T, NX, WS>, sm);
        Prof pf(h, "k_seg_suffix", st);
        k_seg_suffix<T, NX, WS><<<(B + wpb - 1) / wpb, 128, sm, st>>>(B, n, S_all, G, r, Pt, pt, P_out, p_out, ws.fail);
    })
    h->launches = 1;
    return cuda_check("segment suffix launch");
}

template <typename T>
pdilqr_status run_seg_forward(pdilqr_ctx *h, const LqArgs<T> &qp, T *F_out, cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N, n = h->cfg.n, m = h->cfg.m;
    LqWork<T> ws = work<T>(h);
    PDILQR_SEG_DISPATCH({
        const int wpb = 128 / WS;
        const size_t sm = (size_t)wpb * (NX * NX + NX) * sizeof(T);
        set_smem(k_seg_forward<T, NX, WS>, sm);
        Prof pf(h, "k_seg_forward", st);
        k_seg_forward<T, NX, WS><<<(B + wpb - 1) / wpb, 128, sm, st>>>(B, N, n, m, qp, ws, F_out);
    })
    h->launches = 1;
    return cuda_check("segment forward launch");
}

template <typename T>
pdilqr_status run_seg_prefix(pdilqr_ctx *h, const T *F_all, int G, int r, const T *dx0, T *dxs, cudaStream_t st) {
    const int B = h->cfg.batch, n = h->cfg.n;
    PDILQR_SEG_DISPATCH({
        const int wpb = 128 / WS;
        Prof pf(h, "k_seg_prefix", st);
        k_seg_prefix<T, NX, WS><<<(B + wpb - 1) / wpb, 128, 0, st>>>(B, n, F_all, G, r, dx0, dxs);
    })
    h->launches = 1;
    return cuda_check("segment prefix launch");
}
#undef PDILQR_SEG_DISPATCH

template <typename T>
void grid_occupancy(int v, int sms, int &nb, int &nf, int &nk, int &nfk, int &nk2) {
    auto occ = [&](auto kern, size_t smem, int &out) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
        out = std::max(1, per) * sms;
    };
    if (v == V12) { occ(k_scan_bwd_grid<T, 12>, 8 * sizeof(CombineSmem<T, 12>), nb); occ(k_scan_fwd_grid<T, 12>, 8 * sizeof(FwdSmem<T, 12>), nf); }
    else if (v == V4) { occ(k_scan_bwd_grid<T, 4>, 32 * sizeof(CombineSmem<T, 4>), nb); occ(k_scan_fwd_grid<T, 4>, 32 * sizeof(FwdSmem<T, 4>), nf); }
    else if (v == V8) { occ(k_scan_bwd_grid<T, 8>, 16 * sizeof(CombineSmem<T, 8>), nb); occ(k_scan_fwd_grid<T, 8>, 16 * sizeof(FwdSmem<T, 8>), nf); }
    else { occ(k_scan_bwd_grid<T, 16>, 8 * sizeof(CombineSmem<T, 16>), nb); occ(k_scan_fwd_grid<T, 16>, 8 * sizeof(FwdSmem<T, 16>), nf); }
    if (v == V12) occ(k_scan_bwd_ks<T, 12>, 8 * sizeof(CombineSmem<T, 12>), nk);
    else if (v == V4) occ(k_scan_bwd_ks<T, 4>, 32 * sizeof(CombineSmem<T, 4>), nk);
    else if (v == V8) occ(k_scan_bwd_ks<T, 8>, 16 * sizeof(CombineSmem<T, 8>), nk);
    else occ(k_scan_bwd_ks<T, 16>, 8 * sizeof(CombineSmem<T, 16>), nk);
    if (v == V12) occ(k_scan_fwd_ks<T, 12>, 8 * sizeof(FwdSmem<T, 12>), nfk);
    else if (v == V4) occ(k_scan_fwd_ks<T, 4>, 32 * sizeof(FwdSmem<T, 4>), nfk);
    else if (v == V8) occ(k_scan_fwd_ks<T, 8>, 16 * sizeof(FwdSmem<T, 8>), nfk);
    else occ(k_scan_fwd_ks<T, 16>, 8 * sizeof(FwdSmem<T, 16>), nfk);
    if (v == V12) occ(k_scan_bwd_ks2<T, 12>, 4 * sizeof(CombineSmem<T, 12>), nk2);
    else if (v == V16) occ(k_scan_bwd_ks2<T, 16>, 4 * sizeof(CombineSmem<T, 16>), nk2);
}

#define PDILQR_INST_SMALL(T)                                                                                       \
    template pdilqr_status dispatch_lq<T>(pdilqr_ctx *, const LqArgs<T> &, LqOut<T>, int32_t *, const int32_t *,    \
                                          cudaStream_t, bool);                                                     \
    template pdilqr_status run_linearize<T>(pdilqr_ctx *, const pdilqr_iterate *, const LqArgs<T> &, int32_t *,     \
                                            cudaStream_t);                                                         \
    template pdilqr_status run_step<T>(pdilqr_ctx *, pdilqr_iterate *, pdilqr_stats *, pdilqr_dir *, cudaStream_t); \
    template void grid_occupancy<T>(int, int, int &, int &, int &, int &, int &);                               \
    template pdilqr_status run_adjoint<T>(pdilqr_ctx *, const LqArgs<T> &, const LqOut<T> &, const T *, const T *,   \
                                          const T *, const AdjGrad<T> &, int32_t *, cudaStream_t);                   \
    template pdilqr_status run_seg_reduce<T>(pdilqr_ctx *, const LqArgs<T> &, T *, int32_t *, cudaStream_t);         \
    template pdilqr_status run_seg_suffix<T>(pdilqr_ctx *, const T *, int, int, const T *, const T *, T *, T *,      \
                                             cudaStream_t);                                                        \
    template pdilqr_status run_seg_forward<T>(pdilqr_ctx *, const LqArgs<T> &, T *, cudaStream_t);                                      \
    template pdilqr_status run_seg_prefix<T>(pdilqr_ctx *, const T *, int, int, const T *, T *, cudaStream_t);
#if PDILQR_SMALL(0)
PDILQR_INST_SMALL(float)
#endif
#if PDILQR_SMALL(1)
PDILQR_INST_SMALL(double)
#endif
}  // namespace pdq
#endif

#if PDILQR_BIG(0) || PDILQR_BIG(1)
namespace pdq {
// k_big_ric variant: SIMT tiles (5x2 for config-5-like shapes, else 3x3) or tcgen05 (float only)
template <typename T>
using RicKernT = void (*)(LqArgs<T>, int, int, BigDims<T>, BigWork<T>, LqOut<T>, int);
template <typename T>
RicKernT<T> ric_kernel(bool t52, bool ut, bool mm) {
    if constexpr (std::is_same<T, float>::value) {
        if (mm) return k_big_ric<float, 1, 1, false, true>;
        if (ut) return k_big_ric<float, 1, 1, true>;
    }
    (void)ut;
    (void)mm;
    return t52 ? k_big_ric<T, 5, 2> : k_big_ric<T, 3, 3>;
}
template <typename T>
bool ric_use_tc(const pdilqr_ctx *h, int m) {
    return std::is_same<T, float>::value && h->big_tc && ric_smem_bytes_tc(m) <= 227 * 1024;
}

template <typename T>
pdilqr_status run_big(pdilqr_ctx *h, const LqArgs<T> &qp, LqOut<T> out, int32_t *info, cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N, n = h->cfg.n, m = h->cfg.m;
    BigDims<T> d{n, m, ld_of(n), ld_of(m)};
    BigWork<T> ws;
    ws.elems = reinterpret_cast<T *>(h->ws + h->lay.elems);
    ws.Pp = reinterpret_cast<T *>(h->ws + h->lay.Pp);
    ws.Kk = reinterpret_cast<T *>(h->ws + h->lay.Kk);
    ws.tel = reinterpret_cast<T *>(h->ws + h->lay.tel);
    ws.dxw = reinterpret_cast<T *>(h->ws + h->lay.dxw);
    ws.scratch = reinterpret_cast<T *>(h->ws + h->lay.vslots);
    ws.slot = big_slot(n, m);
    ws.fail = reinterpret_cast<int32_t *>(h->ws + h->lay.fail);
    cudaMemsetAsync(ws.fail, 0x7f, (size_t)B * 4, st);
    const size_t ric_smem = ric_smem_bytes(m, (int)sizeof(T));
    if (ric_smem <= kRicSmemMax && !h->big_legacy && !h->lay.elems2) {  // fused Riccati-form fold (big_ric.cuh)
        const bool t52 = n <= 80 && m <= 32 && h->ric_cs == 1;  // config-5-like: 80-row n tiles, 32-wide m tiles
        const bool ut = ric_use_tc<T>(h, m);                      // tcgen05 3xTF32 products (tc.cuh)
        {
            const int tpb = std::min(256, (m + 31) / 32 * 32);  // one thread per row of R
            const int g = (int)std::min<long>((long)148 * (2048 / tpb), (long)B * (N + 1));
            cudaFuncSetAttribute(k_big_rchk<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ric_smem);
            Prof pf(h, "k_big_rchk", st);
            k_big_rchk<T><<<g, tpb, ric_smem, st>>>(qp.R, B, N, m, ws.fail);
        }
        {
            const bool mm = std::is_same<T, float>::value && h->big_mma && !ut;
            auto kern = ric_kernel<T>(t52, ut, mm);
            const size_t smem = ut ? ric_smem_bytes_tc(m) : ric_smem;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (h->ric_cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3((unsigned)(B * h->ric_cs));
            lc.blockDim = dim3(RIC_THREADS);
            lc.dynamicSmemBytes = smem;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)h->ric_cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            Prof pf(h, ut ? "k_big_ric_tc" : mm ? "k_big_ric_mma" : "k_big_ric", st);
            cudaError_t e = cudaLaunchKernelEx(&lc, kern, qp, B, N, d, ws, out, h->ric_cs);
            if (e != cudaSuccess) return fail(PDILQR_ERR_CUDA, "k_big_ric launch (cluster %d): %s", h->ric_cs, cudaGetErrorString(e));
        }
        {
            Prof pf(h, "k_big_roll", st);
            k_big_roll<T><<<B, 256, 0, st>>>(qp.dx0, B, N, d, ws, out.dx);
        }
        {
            Prof pf(h, "k_big_tail", st);
            k_big_tail<T><<<(unsigned)((long)B * (N + 2)), 128, 0, st>>>(B, N, d, ws, out);
        }
        int launches = 4;
        if (info) {
            int32_t *nonfin = reinterpret_cast<int32_t *>(h->ws + h->lay.nonfin);
            cudaMemsetAsync(nonfin, 0, (size_t)B * 4, st);
            Prof pf(h, "k_finalize_info", st);
            k_finalize_info<<<(B + 255) / 256, 256, 0, st>>>(B, ws.fail, nonfin, nullptr, info);
            ++launches;
        }
        h->launches += launches;
        return cuda_check("solve_lq (large, fused) launch");
    }
    const int gpers = (int)std::min<long>((long)kBigPersistent, (long)B * (N + 2));
    // the augmented Gauss-Jordan matrix W lives in shared memory when it fits (n <= ~110 in fp32)
    const size_t kSmemW = 180 * 1024;
    auto wbytes = [&](int rows, int cols) { return (size_t)rows * ld_of(cols) * sizeof(T); };
    {
        const size_t wb = wbytes(m, m + 2 * n + 1);
        const int in = wb <= kSmemW;
        if (in) cudaFuncSetAttribute(k_big_init<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb);  // + static tiles
        Prof pf(h, "k_big_init", st);
        k_big_init<T><<<gpers, BIG_THREADS, in ? wb : 0, st>>>(qp, B, N, d, ws, in);
    }
    int scan_launches = 0;
    if (h->lay.elems2) {
        // leaf_chunk = 1: the paper's reverse associative scan over the N+2 elements,
        // Kogge-Stone levels dl = 1, 2, 4, ... with CTA-level full combines, then the read-out
        const size_t wb = wbytes(n, 3 * n + 1);
        const int in = wb <= kSmemW;
        if (in) cudaFuncSetAttribute(k_bigks_level<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb);
        T *bufs[2] = {ws.elems, reinterpret_cast<T *>(h->ws + h->lay.elems2)};
        int cur = 0;
        const int Lr = N + 2;
        const int gk = (int)std::min<long>((long)kBigPersistent, (long)B * Lr);
        for (int dl = 1; dl < Lr; dl *= 2) {
            Prof pf(h, "k_bigks_level", st);
            k_bigks_level<T><<<gk, BIG_THREADS, in ? wb : 0, st>>>(B, N, dl, d, ws, bufs[cur], bufs[1 - cur], in);
            cur = 1 - cur;
            ++scan_launches;
        }
        Prof pf(h, "k_bigks_readout", st);
        const long tot = (long)B * Lr * (long)(n * d.LD + d.LD);
        k_bigks_readout<T><<<(unsigned)std::min<long>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(B, N, d, bufs[cur], ws.Pp);
        ++scan_launches;
    } else {
        const size_t wb = wbytes(n, 2 * n);
        const int in = wb <= kSmemW;
        if (in) cudaFuncSetAttribute(k_big_fold<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb);  // + static tiles
        Prof pf(h, "k_big_fold", st);
        k_big_fold<T><<<B, BIG_THREADS, in ? wb : 0, st>>>(B, N, d, ws, in);
        ++scan_launches;
    }
    {
        const size_t wb = wbytes(m, m + n + 1);
        const int in = wb <= kSmemW;
        if (in) cudaFuncSetAttribute(k_big_policy<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb);  // + static tiles
        Prof pf(h, "k_big_policy", st);
        k_big_policy<T><<<gpers, BIG_THREADS, in ? wb : 0, st>>>(qp, B, N, d, ws, out, in);
    }
    {
        Prof pf(h, "k_big_fwd", st);
        k_big_fwd<T><<<B, BIG_THREADS, 0, st>>>(qp.dx0, B, N, d, ws, out);
    }
    int launches = 3 + scan_launches;
    if (info) {
        int32_t *nonfin = reinterpret_cast<int32_t *>(h->ws + h->lay.nonfin);
        cudaMemsetAsync(nonfin, 0, (size_t)B * 4, st);
        Prof pf(h, "k_finalize_info", st);
        k_finalize_info<<<(B + 255) / 256, 256, 0, st>>>(B, ws.fail, nonfin, nullptr, info);
        ++launches;
    }
    h->launches += launches;
    return cuda_check("solve_lq (large) launch");
}

template <typename T>
bool ric_cluster_fits(int cs, size_t smem, bool ut) {
    const void *kern = (const void *)ric_kernel<T>(false, ut, false);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)cs);
    lc.blockDim = dim3(RIC_THREADS);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &lc) == cudaSuccess && ncl > 0) return true;
    cudaGetLastError();
    return false;
}
inline MultiConst multi_const(const pdilqr_ctx *h) {
    const auto &mp = h->cfg.multi;
    return MultiConst{mp.n_robots, mp.d_min, mp.weight, mp.sharpness};
}

template <typename T>
pdilqr_status run_multi_linearize(pdilqr_ctx *h, const pdilqr_iterate *it, const LqArgs<T> &outq, int32_t *pre,
                                  cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N;
    cudaMemsetAsync(pre, 0, (size_t)B * 4, st);
    {
        Prof pf(h, "k_multi_linearize", st);
        k_multi_linearize<T><<<(unsigned)((long)B * (N + 2)), MULTI_THREADS, 0, st>>>(h->K, multi_const(h), iter_of<T>(it), B,
                                                                                     N, outq, pre);
    }
    h->launches += 1;
    return cuda_check("multi linearize launch");
}

// One SQP iteration of the centralized OCP: linearise (k_multi_linearize), solve the dense LQ
// subproblem (large-n path or n = 12 path), filter line search + update (k_multi_linesearch).
template <typename T>
pdilqr_status run_multi_step(pdilqr_ctx *h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir, cudaStream_t st) {
    const int B = h->cfg.batch, N = h->cfg.N;
    LqArgs<T> qp = internal_qp<T>(h);
    int32_t *pre = reinterpret_cast<int32_t *>(h->ws + h->lay.pre);
    int32_t *info_tmp = reinterpret_cast<int32_t *>(h->ws + h->lay.info_tmp);
    pdilqr_status s = run_multi_linearize<T>(h, it, qp, pre, st);
    if (s != PDILQR_OK) return s;
    LqOut<T> out;
    if (dir && dir->dx) {
        out = LqOut<T>{(T *)dir->dx, (T *)dir->du, (T *)dir->dlam, (T *)dir->K, (T *)dir->k};
    } else {
        out = LqOut<T>{reinterpret_cast<T *>(h->ws + h->lay.dir[0]), reinterpret_cast<T *>(h->ws + h->lay.dir[1]),
                       reinterpret_cast<T *>(h->ws + h->lay.dir[2]), nullptr, nullptr};
    }
    s = dispatch_lq<T>(h, qp, out, info_tmp, nullptr, st);
    if (s != PDILQR_OK) return s;
    LsOut<T> so{(T *)stats->cost, (T *)stats->theta, (T *)stats->alpha, stats->accepted, stats->info};
    {
        Prof pf(h, "k_multi_linesearch", st);
        k_multi_linesearch<T><<<B, MULTI_THREADS, 0, st>>>(h->K, multi_const(h), iter_of<T>(it), B, N, out.dx, out.du,
                                                           out.dlam, info_tmp, pre, so);
    }
    h->launches += 1;
    return cuda_check("multi step launch");
}

#if PDILQR_BIG(0)
template pdilqr_status run_multi_linearize<float>(pdilqr_ctx *, const pdilqr_iterate *, const LqArgs<float> &, int32_t *,
                                                  cudaStream_t);
template pdilqr_status run_multi_step<float>(pdilqr_ctx *, pdilqr_iterate *, pdilqr_stats *, pdilqr_dir *, cudaStream_t);
#endif
#if PDILQR_BIG(1)
template pdilqr_status run_multi_linearize<double>(pdilqr_ctx *, const pdilqr_iterate *, const LqArgs<double> &,
                                                   int32_t *, cudaStream_t);
template pdilqr_status run_multi_step<double>(pdilqr_ctx *, pdilqr_iterate *, pdilqr_stats *, pdilqr_dir *, cudaStream_t);
#endif
#if PDILQR_BIG(0)
cudaError_t debug_tc_gemm(int M, int N, int K, int ta, int tb, const float *A, int lda, const float *Bm, int ldb,
                          const float *Cin, float *C, cudaStream_t st) {
    const size_t smem = sizeof(TcSmem);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, 256, smem, st>>>(M, N, K, A, lda, Bm, ldb, Cin, C);
    };
    if (ta && tb) go(k_tc_gemm_test<true, true>);
    else if (ta) go(k_tc_gemm_test<true, false>);
    else if (tb) go(k_tc_gemm_test<false, true>);
    else go(k_tc_gemm_test<false, false>);
    return cudaGetLastError();
}
template pdilqr_status run_big<float>(pdilqr_ctx *, const LqArgs<float> &, LqOut<float>, int32_t *, cudaStream_t);
template bool ric_cluster_fits<float>(int, size_t, bool);
#endif
#if PDILQR_BIG(1)
template pdilqr_status run_big<double>(pdilqr_ctx *, const LqArgs<double> &, LqOut<double>, int32_t *, cudaStream_t);
template bool ric_cluster_fits<double>(int, size_t, bool);
#endif
}  // namespace pdq
#endif

#if PDILQR_HOST
namespace pdq {
thread_local std::string g_err = "ok";
}
using pdq::dispatch_lq;
using pdq::run_linearize;
using pdq::run_step;

namespace {
void inv3(const double *M, double *Mi) {
    const double a = M[0], b = M[1], c = M[2], d = M[3], e = M[4], f = M[5], g = M[6], hh = M[7], i = M[8];
    const double det = a * (e * i - f * hh) - b * (d * i - f * g) + c * (d * hh - e * g);
    Mi[0] = (e * i - f * hh) / det; Mi[1] = (c * hh - b * i) / det; Mi[2] = (b * f - c * e) / det;
    Mi[3] = (f * g - d * i) / det;  Mi[4] = (a * i - c * g) / det;  Mi[5] = (c * d - a * f) / det;
    Mi[6] = (d * hh - e * g) / det; Mi[7] = (b * g - a * hh) / det; Mi[8] = (a * e - b * d) / det;
}

}  // namespace

// ==================================================================================== C ABI
extern "C" {

int32_t pdilqr_abi_version(void) { return PDILQR_ABI_VERSION; }

const char *pdilqr_last_error(void) { return g_err.c_str(); }

int32_t pdilqr_last_launch_count(pdilqr_handle h) { return h ? h->launches : 0; }

pdilqr_status pdilqr_workspace_bytes(const pdilqr_config *cfg, size_t *bytes) {
    Variant v;
    int NX, NU;
    pdilqr_status s = check_cfg(cfg, v, NX, NU);
    if (s != PDILQR_OK) return s;
    if (!bytes) return fail(PDILQR_ERR_INVALID_ARG, "bytes is NULL");
    int Jb, Pv, Jf, Pf;
    const int esz = cfg->dtype == PDILQR_F32 ? 4 : 8;
    *bytes = make_layout(cfg, NX, NU, esz, default_chunk(cfg), Jb, Pv, Jf, Pf).total;
    return PDILQR_OK;
}

pdilqr_status pdilqr_create(const pdilqr_config *cfg, int device, void *workspace, size_t bytes, pdilqr_handle *out) {
    Variant v;
    int NX, NU;
    pdilqr_status s = check_cfg(cfg, v, NX, NU);
    if (s != PDILQR_OK) return s;
    if (!out) return fail(PDILQR_ERR_INVALID_ARG, "out is NULL");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(PDILQR_ERR_CUDA, "no CUDA device %d (count %d)", device, ndev);
    const int esz = cfg->dtype == PDILQR_F32 ? 4 : 8;
    const int chunk = default_chunk(cfg);
    int Jb, Pv, Jf, Pf;
    Layout L = make_layout(cfg, NX, NU, esz, chunk, Jb, Pv, Jf, Pf);
    if (!workspace || bytes < L.total)
        return fail(PDILQR_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", bytes, L.total);
    if (reinterpret_cast<uintptr_t>(workspace) % kAlign)
        return fail(PDILQR_ERR_WORKSPACE, "workspace must be %zu-byte aligned", kAlign);
    pdilqr_ctx *h = new (std::nothrow) pdilqr_ctx();
    if (!h) return fail(PDILQR_ERR_INVALID_ARG, "out of host memory");
    h->cfg = *cfg;
    if (h->cfg.n_alpha == 0) h->cfg.n_alpha = 10;
    if (h->cfg.armijo_c1 == 0) h->cfg.armijo_c1 = 1e-4;
    if (h->cfg.theta_max <= 0) h->cfg.theta_max = 1e-2 * (cfg->N + 1);
    h->device = device;
    h->var = v;
    h->NX = NX;
    h->NU = NU;
    h->esz = esz;
    h->chunk = chunk;
    h->Jb = Jb; h->Pv = Pv; h->Jf = Jf; h->Pf = Pf;
    h->ws = static_cast<char *>(workspace);
    h->ws_bytes = bytes;
    {   // defined contents once: padded lanes and unused tree slots are then never uninitialised reads
        // (compute-sanitizer initcheck); setup only, not on the hot path
        DeviceGuard g0(device);
        if (cudaMemset(workspace, 0, L.total) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
            delete h;
            return fail(PDILQR_ERR_CUDA, "workspace initialisation failed: %s", cudaGetErrorString(cudaGetLastError()));
        }
    }
    h->lay = L;
    h->launches = 0;
    SrbdConst &K = h->K;
    std::memset(&K, 0, sizeof K);
    const pdilqr_srbd_params &p = cfg->srbd;
    K.dt = p.dt; K.mass = p.mass;
    for (int k = 0; k < 9; ++k) K.I[k] = p.inertia[k];
    inv3(p.inertia, K.Iinv);
    for (int k = 0; k < 3; ++k) K.g[k] = p.gravity[k];
    for (int k = 0; k < 12; ++k) { K.wx[k] = p.w_x[k]; K.wxt[k] = p.w_x_term[k]; }
    K.wu_st = p.w_u_stance; K.wu_sw = p.w_u_swing;
    K.mu = p.mu_friction; K.fmin = p.f_min; K.fmax = p.f_max; K.bmu = p.barrier_mu; K.bdelta = p.barrier_delta;
    K.imass = 1.0 / p.mass;
    K.ibd = 1.0 / p.barrier_delta;
    K.ibd2 = 1.0 / (p.barrier_delta * p.barrier_delta);
    K.theta_max = h->cfg.theta_max; K.c1 = h->cfg.armijo_c1; K.n_alpha = h->cfg.n_alpha;
    if (const char *e = std::getenv("PDILQR_OCC_FOLD")) h->occ_fold = std::atoi(e);  // tuning knobs
    if (const char *e = std::getenv("PDILQR_OCC_LS")) h->occ_ls = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FOLD_TPB")) h->fold_tpb = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FUSED")) h->fused = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_LINREC")) h->linrec = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FOLD_W")) h->fold_w = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FOLD_MODE")) h->fold_mode = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FOLD_NW")) h->fold_nw = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FOLD_CP")) h->fold_cp = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_LIN_STAGED")) h->lin_staged = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_ELEM_R2")) h->elem_r2 = std::atoi(e);
    if (const char *e = std::getenv("PDILQR_FAULT_COMBINE")) h->fault_combine = std::atoi(e) != 0;
    if (const char *e = std::getenv("PDILQR_NVTX")) h->nvtx = std::atoi(e) != 0;
    if (v == VBIG) {  // large path: cluster size of k_big_ric (CTAs per instance) so that B * CS fills the SMs
        if (const char *e = std::getenv("PDILQR_BIG_LEGACY")) h->big_legacy = std::atoi(e) != 0;
        DeviceGuard g(device);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        int cs = 1;
        while (cs < 16 && (long)cfg->batch * cs * 2 <= sms) cs *= 2;
        if (const char *e = std::getenv("PDILQR_BIG_CS")) cs = std::max(1, std::min(16, std::atoi(e)));
        if (const char *e = std::getenv("PDILQR_BIG_TC")) h->big_tc = std::atoi(e) != 0;
        if (const char *e = std::getenv("PDILQR_BIG_MMA")) h->big_mma = std::atoi(e) != 0;
        const bool ut = esz == 4 && h->big_tc && ric_smem_bytes_tc(cfg->m) <= 227 * 1024;
        const size_t smem = ut ? ric_smem_bytes_tc(cfg->m) : ric_smem_bytes(cfg->m, esz);
        while (cs > 1 && ric_smem_bytes(cfg->m, esz) <= kRicSmemMax) {  // the device must co-schedule a whole cluster
            if (esz == 4 ? pdq::ric_cluster_fits<float>(cs, smem, ut) : pdq::ric_cluster_fits<double>(cs, smem, false)) break;
            cs /= 2;
        }
        h->ric_cs = cs;
    }
    // latency regime: few instances -> spread every tree level over all SMs (cooperative launch)
    h->grid_scan = cfg->batch < 148 && (Jb > 1 || Jf > 1);
    if (const char *e = std::getenv("PDILQR_GRID_SCAN")) h->grid_scan = std::atoi(e) != 0 && (Jb > 1 || Jf > 1);
    if (h->grid_scan) {
        DeviceGuard g(device);
        int sms = 148, nb = 0, nf = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        int nk = 0, nfk = 0, nk2 = 0;
        if (esz == 4) pdq::grid_occupancy<float>(v, sms, nb, nf, nk, nfk, nk2);
        else pdq::grid_occupancy<double>(v, sms, nb, nf, nk, nfk, nk2);
        h->coop_bwd = nb;
        h->coop_fwd = nf;
        h->coop_ks = nk;
        h->coop_fks = nfk;
        h->coop_ks2 = nk2;
        if (const char *e = std::getenv("PDILQR_KS_SPLIT")) h->ks_split = std::atoi(e) != 0;
        // Kogge-Stone when every level of the pure tree fits in one wave of resident workers
        const int wpb = 128 / worker_width(NX);
        h->ks_bwd = chunk == 1 && (long)cfg->batch * (cfg->N + 2) <= (long)nk * wpb;
        if (const char *e = std::getenv("PDILQR_SCAN_KS")) h->ks_bwd = chunk == 1 && std::atoi(e) != 0;
    }
    *out = h;
    return PDILQR_OK;
}

pdilqr_status pdilqr_destroy(pdilqr_handle h) {
    if (h) {
        for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    }
    delete h;
    return PDILQR_OK;
}

pdilqr_status pdilqr_profile(pdilqr_handle h, int32_t enable) {
    if (!h) return fail(PDILQR_ERR_INVALID_ARG, "NULL handle");
    h->prof = enable != 0;
    h->recs.clear();
    h->ev_used = 0;
    return PDILQR_OK;
}

int32_t pdilqr_profile_read(pdilqr_handle h, int32_t max, const char **names, int32_t *launches, double *total_ms) {
    if (!h) return -1;
    DeviceGuard g(h->device);
    std::vector<const char *> nm;
    std::vector<int32_t> cnt;
    std::vector<double> tot;
    for (const ProfRec &r : h->recs) {
        cudaEventSynchronize(r.stop);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.start, r.stop);
        size_t k = 0;
        while (k < nm.size() && std::strcmp(nm[k], r.name) != 0) ++k;
        if (k == nm.size()) { nm.push_back(r.name); cnt.push_back(0); tot.push_back(0); }
        cnt[k] += 1;
        tot[k] += ms;
    }
    const int32_t n = (int32_t)nm.size();
    for (int32_t k = 0; k < n && k < max; ++k) {
        if (names) names[k] = nm[k];
        if (launches) launches[k] = cnt[k];
        if (total_ms) total_ms[k] = tot[k];
    }
    h->recs.clear();
    h->ev_used = 0;
    return n;
}

pdilqr_status pdilqr_solve_lq(pdilqr_handle h, const pdilqr_lq *qp, pdilqr_dir *dir, int32_t *info, void *stream) {
    if (!h || !qp || !dir) return fail(PDILQR_ERR_INVALID_ARG, "NULL handle, qp or dir");
    const void *ptrs[] = {qp->A, qp->Bm, qp->c, qp->Q, qp->R, qp->S, qp->q, qp->r, qp->P_term, qp->p_term, qp->dx0,
                          dir->dx, dir->du, dir->dlam};
    for (const void *p : ptrs) {
        if (!p) return fail(PDILQR_ERR_INVALID_ARG, "NULL array in qp / dir");
        if (!aligned16(p)) return fail(PDILQR_ERR_INVALID_ARG, "arrays must be 16-byte aligned");
    }
    DeviceGuard g(h->device);
    h->launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->cfg.dtype == PDILQR_F32) {
        LqArgs<float> a{(const float *)qp->A, (const float *)qp->Bm, (const float *)qp->c, (const float *)qp->Q,
                        (const float *)qp->R, (const float *)qp->S, (const float *)qp->q, (const float *)qp->r,
                        (const float *)qp->P_term, (const float *)qp->p_term, (const float *)qp->dx0};
        LqOut<float> o{(float *)dir->dx, (float *)dir->du, (float *)dir->dlam, (float *)dir->K, (float *)dir->k};
        return dispatch_lq<float>(h, a, o, info, nullptr, st);
    }
    LqArgs<double> a{(const double *)qp->A, (const double *)qp->Bm, (const double *)qp->c, (const double *)qp->Q,
                     (const double *)qp->R, (const double *)qp->S, (const double *)qp->q, (const double *)qp->r,
                     (const double *)qp->P_term, (const double *)qp->p_term, (const double *)qp->dx0};
    LqOut<double> o{(double *)dir->dx, (double *)dir->du, (double *)dir->dlam, (double *)dir->K, (double *)dir->k};
    return dispatch_lq<double>(h, a, o, info, nullptr, st);
}

pdilqr_status pdilqr_solve_lq_adjoint(pdilqr_handle h, const pdilqr_lq *qp, const pdilqr_dir *sol,
                                      const pdilqr_dir *gsol, pdilqr_lq_grad *grad, int32_t *info, void *stream) {
    if (!h || !qp || !sol || !grad) return fail(PDILQR_ERR_INVALID_ARG, "NULL handle, qp, sol or grad");
    const void *ptrs[] = {qp->A, qp->Bm, qp->Q, qp->R, qp->S, qp->P_term, sol->dx, sol->du, sol->dlam};
    for (const void *p : ptrs) {
        if (!p) return fail(PDILQR_ERR_INVALID_ARG, "NULL matrix in qp or NULL array in sol");
        if (!aligned16(p)) return fail(PDILQR_ERR_INVALID_ARG, "arrays must be 16-byte aligned");
    }
    DeviceGuard g(h->device);
    h->launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto run = [&](auto zero) {
        using T = decltype(zero);
        LqArgs<T> a{(const T *)qp->A, (const T *)qp->Bm, nullptr, (const T *)qp->Q, (const T *)qp->R, (const T *)qp->S,
                    nullptr, nullptr, (const T *)qp->P_term, nullptr, nullptr};
        LqOut<T> z{(T *)sol->dx, (T *)sol->du, (T *)sol->dlam, nullptr, nullptr};
        AdjGrad<T> gr{(T *)grad->A, (T *)grad->Bm, (T *)grad->c, (T *)grad->Q, (T *)grad->R, (T *)grad->S,
                      (T *)grad->q, (T *)grad->r, (T *)grad->P_term, (T *)grad->p_term, (T *)grad->dx0};
        const T *gx = gsol ? (const T *)gsol->dx : nullptr, *gu = gsol ? (const T *)gsol->du : nullptr,
                *gl = gsol ? (const T *)gsol->dlam : nullptr;
        return pdq::run_adjoint<T>(h, a, z, gx, gu, gl, gr, info, st);
    };
    return h->cfg.dtype == PDILQR_F32 ? run(0.0f) : run(0.0);
}

pdilqr_status pdilqr_lq_segment_reduce(pdilqr_handle h, const pdilqr_lq *qp, void *S_out, int32_t *info, void *stream) {
    if (!h || !qp || !S_out) return fail(PDILQR_ERR_INVALID_ARG, "NULL handle, qp or S_out");
    if (h->cfg.model != PDILQR_MODEL_LQ) return fail(PDILQR_ERR_UNSUPPORTED, "horizon sharding serves LQ handles");
    const void *ptrs[] = {qp->A, qp->Bm, qp->c, qp->Q, qp->R, qp->S, qp->q, qp->r, qp->P_term, qp->p_term, qp->dx0};
    for (const void *p : ptrs)
        if (!p || !aligned16(p)) return fail(PDILQR_ERR_INVALID_ARG, "NULL or misaligned array in qp");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto run = [&](auto zero) {
        using T = decltype(zero);
        LqArgs<T> a{(const T *)qp->A, (const T *)qp->Bm, (const T *)qp->c, (const T *)qp->Q, (const T *)qp->R,
                    (const T *)qp->S, (const T *)qp->q, (const T *)qp->r, (const T *)qp->P_term, (const T *)qp->p_term,
                    (const T *)qp->dx0};
        return pdq::run_seg_reduce<T>(h, a, (T *)S_out, info, st);
    };
    return h->cfg.dtype == PDILQR_F32 ? run(0.0f) : run(0.0);
}

pdilqr_status pdilqr_lq_segment_suffix(pdilqr_handle h, const void *S_all, int32_t G, int32_t r, const void *P_term,
                                       const void *p_term, void *P_out, void *p_out, void *stream) {
    if (!h || !S_all || !P_term || !p_term || !P_out || !p_out) return fail(PDILQR_ERR_INVALID_ARG, "NULL argument");
    if (G < 1 || r < 0 || r >= G) return fail(PDILQR_ERR_INVALID_ARG, "need 0 <= r < G");
    if (h->cfg.model != PDILQR_MODEL_LQ) return fail(PDILQR_ERR_UNSUPPORTED, "horizon sharding serves LQ handles");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->cfg.dtype == PDILQR_F32)
        return pdq::run_seg_suffix<float>(h, (const float *)S_all, G, r, (const float *)P_term, (const float *)p_term,
                                          (float *)P_out, (float *)p_out, st);
    return pdq::run_seg_suffix<double>(h, (const double *)S_all, G, r, (const double *)P_term, (const double *)p_term,
                                       (double *)P_out, (double *)p_out, st);
}

pdilqr_status pdilqr_lq_segment_forward(pdilqr_handle h, const pdilqr_lq *qp, void *F_out, void *stream) {
    if (!h || !qp || !F_out || !qp->A || !qp->Bm || !qp->c) return fail(PDILQR_ERR_INVALID_ARG, "NULL argument");
    if (h->cfg.model != PDILQR_MODEL_LQ) return fail(PDILQR_ERR_UNSUPPORTED, "horizon sharding serves LQ handles");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto run = [&](auto zero) {
        using T = decltype(zero);
        LqArgs<T> a{(const T *)qp->A, (const T *)qp->Bm, (const T *)qp->c, nullptr, nullptr, nullptr, nullptr, nullptr,
                    nullptr, nullptr, nullptr};
        return pdq::run_seg_forward<T>(h, a, (T *)F_out, st);
    };
    return h->cfg.dtype == PDILQR_F32 ? run(0.0f) : run(0.0);
}

pdilqr_status pdilqr_lq_segment_prefix(pdilqr_handle h, const void *F_all, int32_t G, int32_t r, const void *dx0,
                                       void *dxs_out, void *stream) {
    if (!h || !F_all || !dx0 || !dxs_out) return fail(PDILQR_ERR_INVALID_ARG, "NULL argument");
    if (G < 1 || r < 0 || r >= G) return fail(PDILQR_ERR_INVALID_ARG, "need 0 <= r < G");
    if (h->cfg.model != PDILQR_MODEL_LQ) return fail(PDILQR_ERR_UNSUPPORTED, "horizon sharding serves LQ handles");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->cfg.dtype == PDILQR_F32)
        return pdq::run_seg_prefix<float>(h, (const float *)F_all, G, r, (const float *)dx0, (float *)dxs_out, st);
    return pdq::run_seg_prefix<double>(h, (const double *)F_all, G, r, (const double *)dx0, (double *)dxs_out, st);
}

pdilqr_status pdilqr_debug_tc_gemm(int32_t M, int32_t N, int32_t K, int32_t trans_a, int32_t trans_b, const float *A,
                                   int32_t lda, const float *Bm, int32_t ldb, const float *Cin, float *C, void *stream) {
    if (M < 1 || N < 1 || K < 1 || M > 256 || N > 256) return fail(PDILQR_ERR_DIM, "debug_tc_gemm: 1 <= M, N <= 256, K >= 1");
    if (!A || !Bm || !C) return fail(PDILQR_ERR_INVALID_ARG, "debug_tc_gemm: NULL array");
    cudaError_t e = pdq::debug_tc_gemm(M, N, K, trans_a, trans_b, A, lda, Bm, ldb, Cin, C, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? PDILQR_OK : fail(PDILQR_ERR_CUDA, "debug_tc_gemm: %s", cudaGetErrorString(e));
}

static pdilqr_status check_iter(pdilqr_handle h, const pdilqr_iterate *it) {
    if (!h || !it) return fail(PDILQR_ERR_INVALID_ARG, "NULL handle or iterate");
    if (h->cfg.model == PDILQR_MODEL_LQ) return fail(PDILQR_ERR_UNSUPPORTED, "handle was not created for a built-in model");
    const void *ptrs[] = {it->x, it->u, it->lam, it->x0, it->x_ref, it->contact, it->feet};
    for (const void *p : ptrs)
        if (!p) return fail(PDILQR_ERR_INVALID_ARG, "NULL array in iterate");
    const void *al[] = {it->x, it->u, it->lam, it->x0, it->x_ref, it->feet};
    for (const void *p : al)
        if (!aligned16(p)) return fail(PDILQR_ERR_INVALID_ARG, "iterate arrays must be 16-byte aligned");
    if (it->u_ref && !aligned16(it->u_ref)) return fail(PDILQR_ERR_INVALID_ARG, "u_ref must be 16-byte aligned");
    return PDILQR_OK;
}

pdilqr_status pdilqr_linearize(pdilqr_handle h, const pdilqr_iterate *it, pdilqr_lq_buf *out, int32_t *info,
                               void *stream) {
    pdilqr_status s = check_iter(h, it);
    if (s != PDILQR_OK) return s;
    if (!out) return fail(PDILQR_ERR_INVALID_ARG, "NULL out");
    void *ptrs[] = {out->A, out->Bm, out->c, out->Q, out->R, out->S, out->q, out->r, out->P_term, out->p_term, out->dx0};
    for (void *p : ptrs)
        if (!p || !aligned16(p)) return fail(PDILQR_ERR_INVALID_ARG, "output arrays must be non-NULL and 16-byte aligned");
    DeviceGuard g(h->device);
    h->launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t *pre = info ? info : reinterpret_cast<int32_t *>(h->ws + h->lay.pre);
    if (h->cfg.dtype == PDILQR_F32) {
        LqArgs<float> o{(float *)out->A, (float *)out->Bm, (float *)out->c, (float *)out->Q, (float *)out->R,
                        (float *)out->S, (float *)out->q, (float *)out->r, (float *)out->P_term, (float *)out->p_term,
                        (float *)out->dx0};
        if (h->cfg.model == PDILQR_MODEL_MULTI_SRBD) return pdq::run_multi_linearize<float>(h, it, o, pre, st);
        return run_linearize<float>(h, it, o, pre, st);
    }
    LqArgs<double> o{(double *)out->A, (double *)out->Bm, (double *)out->c, (double *)out->Q, (double *)out->R,
                     (double *)out->S, (double *)out->q, (double *)out->r, (double *)out->P_term, (double *)out->p_term,
                     (double *)out->dx0};
    if (h->cfg.model == PDILQR_MODEL_MULTI_SRBD) return pdq::run_multi_linearize<double>(h, it, o, pre, st);
    return run_linearize<double>(h, it, o, pre, st);
}

pdilqr_status pdilqr_step(pdilqr_handle h, pdilqr_iterate *it, pdilqr_stats *stats, pdilqr_dir *dir, void *stream) {
    pdilqr_status s = check_iter(h, it);
    if (s != PDILQR_OK) return s;
    if (!stats || !stats->cost || !stats->theta || !stats->alpha || !stats->accepted || !stats->info)
        return fail(PDILQR_ERR_INVALID_ARG, "NULL stats array");
    if (dir && dir->dx && (!dir->du || !dir->dlam)) return fail(PDILQR_ERR_INVALID_ARG, "dir needs dx, du and dlam");
    DeviceGuard g(h->device);
    h->launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->cfg.model == PDILQR_MODEL_MULTI_SRBD)
        return h->cfg.dtype == PDILQR_F32 ? pdq::run_multi_step<float>(h, it, stats, dir, st)
                                          : pdq::run_multi_step<double>(h, it, stats, dir, st);
    if (h->cfg.dtype == PDILQR_F32) return run_step<float>(h, it, stats, dir, st);
    return run_step<double>(h, it, stats, dir, st);
}

pdilqr_status pdilqr_solve(pdilqr_handle h, pdilqr_iterate *it, int32_t max_iters, double tol, pdilqr_stats *stats,
                           int32_t *iters, int32_t *iters_run, void *stream) {
    pdilqr_status s = check_iter(h, it);
    if (s == PDILQR_OK && h->cfg.model != PDILQR_MODEL_SRBD)
        s = fail(PDILQR_ERR_UNSUPPORTED, "solve / shift / plant / tick_host serve single-robot SRBD handles");
    if (s != PDILQR_OK) return s;
    if (!stats || !stats->cost || !stats->theta || !stats->alpha || !stats->accepted || !stats->info)
        return fail(PDILQR_ERR_INVALID_ARG, "NULL stats array");
    if (max_iters < 0 || !(tol >= 0.0)) return fail(PDILQR_ERR_INVALID_ARG, "max_iters < 0 or tol < 0");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = h->cfg.batch;
    int32_t *conv = reinterpret_cast<int32_t *>(h->ws + h->lay.conv);
    int32_t *active = reinterpret_cast<int32_t *>(h->ws + h->lay.active);
    double *rho = reinterpret_cast<double *>(h->ws + h->lay.rho);
    cudaMemsetAsync(conv, 0, (size_t)B * 4, st);
    cudaMemsetAsync(rho, 0, (size_t)B * 8, st);
    int total = 0, run = 0;
    for (int k = 1; k <= max_iters; ++k) {
        cudaMemsetAsync(active, 0, 4, st);
        h->sc_conv = conv;
        h->sc_active = active;
        h->sc_rho = rho;
        h->sc_tol = tol;
        h->sc_iter = k;
        h->launches = 0;
        s = (h->cfg.dtype == PDILQR_F32) ? run_step<float>(h, it, stats, nullptr, st) : run_step<double>(h, it, stats, nullptr, st);
        h->sc_conv = h->sc_active = nullptr;
        h->sc_rho = nullptr;
        total += h->launches;
        if (s != PDILQR_OK) return s;
        run = k;
        int32_t act = 0;
        cudaMemcpyAsync(&act, active, 4, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check("solve sync");
        if (act == 0) break;
    }
    if (iters) cudaMemcpyAsync(iters, conv, (size_t)B * 4, cudaMemcpyDeviceToDevice, st);
    if (iters_run) *iters_run = run;
    h->launches = total;
    return cuda_check("solve");
}

pdilqr_status pdilqr_shift(pdilqr_handle h, pdilqr_iterate *it, void *stream) {
    pdilqr_status s = check_iter(h, it);
    if (s == PDILQR_OK && h->cfg.model != PDILQR_MODEL_SRBD)
        s = fail(PDILQR_ERR_UNSUPPORTED, "solve / shift / plant / tick_host serve single-robot SRBD handles");
    if (s != PDILQR_OK) return s;
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = h->cfg.batch, N = h->cfg.N;
    const long tot = (long)B * 36;
    h->launches = 1;
    if (h->cfg.dtype == PDILQR_F32) {
        Prof pf(h, "k_srbd_shift", st);
        k_srbd_shift<float><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(iter_of<float>(it), B, N);
    } else {
        Prof pf(h, "k_srbd_shift", st);
        k_srbd_shift<double><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(iter_of<double>(it), B, N);
    }
    return cuda_check("shift launch");
}

pdilqr_status pdilqr_srbd_plant(pdilqr_handle h, const pdilqr_iterate *it, void *x_plant, const void *u_hold,
                                const void *ext_force, double dt, int32_t substeps, void *stream) {
    pdilqr_status s = check_iter(h, it);
    if (s == PDILQR_OK && h->cfg.model != PDILQR_MODEL_SRBD)
        s = fail(PDILQR_ERR_UNSUPPORTED, "solve / shift / plant / tick_host serve single-robot SRBD handles");
    if (s != PDILQR_OK) return s;
    if (!x_plant || !u_hold || substeps < 1 || !(dt >= 0)) return fail(PDILQR_ERR_INVALID_ARG, "invalid plant arguments");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = h->cfg.batch, N = h->cfg.N;
    h->launches = 1;
    if (h->cfg.dtype == PDILQR_F32) {
        Prof pf(h, "k_srbd_plant", st);
        k_srbd_plant<float><<<(B + 127) / 128, 128, 0, st>>>(h->K, iter_of<float>(it), B, N, (float *)x_plant,
                                                            (const float *)u_hold, (const float *)ext_force, (float)dt, substeps);
    } else {
        Prof pf(h, "k_srbd_plant", st);
        k_srbd_plant<double><<<(B + 127) / 128, 128, 0, st>>>(h->K, iter_of<double>(it), B, N, (double *)x_plant,
                                                             (const double *)u_hold, (const double *)ext_force, dt, substeps);
    }
    return cuda_check("plant launch");
}

pdilqr_status pdilqr_tick_host(pdilqr_handle h, pdilqr_iterate *it, const void *x0_host, void *u0_host, void *cost_host,
                               void *theta_host, void *alpha_host, int32_t *accepted_host, int32_t *info_host,
                               void *stream) {
    pdilqr_status s = check_iter(h, it);
    if (s == PDILQR_OK && h->cfg.model != PDILQR_MODEL_SRBD)
        s = fail(PDILQR_ERR_UNSUPPORTED, "solve / shift / plant / tick_host serve single-robot SRBD handles");
    if (s != PDILQR_OK) return s;
    if (!x0_host || !u0_host) return fail(PDILQR_ERR_INVALID_ARG, "NULL host buffer");
    DeviceGuard g(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t B = h->cfg.batch, N = h->cfg.N, es = h->esz;
    cudaMemcpyAsync(const_cast<void *>(it->x0), x0_host, B * 12 * es, cudaMemcpyHostToDevice, st);
    char *sp = h->ws + h->lay.stats;  // device stats scratch of this handle
    pdilqr_stats ds;
    ds.cost = sp;
    ds.theta = sp + B * es;
    ds.alpha = sp + 2 * B * es;
    ds.accepted = reinterpret_cast<int32_t *>(sp + 3 * B * es);
    ds.info = reinterpret_cast<int32_t *>(sp + 3 * B * es + B * 4);
    h->launches = 0;
    s = (h->cfg.dtype == PDILQR_F32) ? run_step<float>(h, it, &ds, nullptr, st) : run_step<double>(h, it, &ds, nullptr, st);
    if (s != PDILQR_OK) return s;
    cudaMemcpy2DAsync(u0_host, 12 * es, it->u, (N + 1) * 12 * es, 12 * es, B, cudaMemcpyDeviceToHost, st);
    if (cost_host) cudaMemcpyAsync(cost_host, ds.cost, B * es, cudaMemcpyDeviceToHost, st);
    if (theta_host) cudaMemcpyAsync(theta_host, ds.theta, B * es, cudaMemcpyDeviceToHost, st);
    if (alpha_host) cudaMemcpyAsync(alpha_host, ds.alpha, B * es, cudaMemcpyDeviceToHost, st);
    if (accepted_host) cudaMemcpyAsync(accepted_host, ds.accepted, B * 4, cudaMemcpyDeviceToHost, st);
    if (info_host) cudaMemcpyAsync(info_host, ds.info, B * 4, cudaMemcpyDeviceToHost, st);
    return cuda_check("tick_host");
}

}  // extern "C"
#endif  // PDILQR_HOST
