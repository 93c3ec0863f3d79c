// tc.cuh -- 5th-generation tensor cores (tcgen05) for the large-n products of the Riccati-form fold
// (big_ric.cuh), FP32-accurate by the 3xTF32 split (plain TF32 fails the 1e-4
// parity bar at n = 74 / 192, 3xTF32 passes it).
//
//   x = hi + lo,  hi = x with the low 13 mantissa bits cleared (exactly a TF32 value), lo = x - hi
//   (exact in FP32, |lo| < 2^-10 |x|);  A B ~ A_hi B_hi + A_hi B_lo + A_lo B_hi   (the dropped
//   A_lo B_lo and the TF32 rounding of lo are O(2^-20) relative), accumulated in FP32 in TMEM.
//
// One CTA computes output tiles of 128 rows x NT (<= 128) columns: the operand panels of KC = 16
// k-values are staged by all threads from global memory (L2-resident per instance) into shared
// memory in the canonical K-major no-swizzle UMMA layout (8-row x 16-byte core matrices), split
// into hi / lo on the way; one elected thread issues tcgen05.mma.cta_group::1.kind::tf32
// (M = 128, N = NT, K = 8 per instruction, 3 per k-step) with the accumulator in tensor memory,
// and commits to an mbarrier; the epilogue reads the accumulator with tcgen05.ld (32 lanes x 32-bit,
// 16 columns per load; warp w owns TMEM lanes 32 (w % 4) ..), adds Cin and stores C.
// The panel buffers are double-buffered: the threads stage panel k+1 while the tensor core works on
// panel k.
#pragma once

#include <cstdint>

namespace pdilqr {

constexpr int TC_M = 128;        // UMMA M (one TMEM lane per output row)
constexpr int TC_KC = 16;        // k-values per staged panel (2 UMMA k-steps of 8)
constexpr int TC_NMAX = 128;     // max UMMA N per tile (TMEM columns per accumulator)
constexpr int TC_PANEL = TC_M * TC_KC;  // floats per operand panel (A: 128 rows; B: <= 128 rows)

struct TcSmem {
    float a_hi[2][TC_PANEL], a_lo[2][TC_PANEL], b_hi[2][TC_PANEL], b_lo[2][TC_PANEL];
    unsigned long long mbar[2];
    uint32_t tmem_base;
};

// Per-thread mbarrier phase bits (bit b: parity of the next completion of mbar[b]); every thread
// of the CTA runs the same sequence of waits, so the copies stay identical.
struct TcPhase {
    uint32_t bits = 0;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor, K-major, no swizzle (canonical layout ((8, m), 2) : ((16 B, SBO), LBO)):
// start address, leading byte offset (between the two 16-byte K chunks of one k-step), stride byte
// offset (between 8-row groups), version 1 (sm_100), layout type 0.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;
}

// Instruction descriptor of kind::tf32: D format F32 (bits 4-5 = 1), A, B format TF32 (bits 7-9,
// 10-12 = 2), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
__device__ __forceinline__ uint32_t umma_idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        :
        : "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(unsigned long long *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(unsigned long long *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMEM allocation by warp 0 (ncols: power of two >= 32); the base address lands in sm.tmem_base.
__device__ __forceinline__ void tc_alloc(TcSmem &sm, uint32_t ncols) {
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
}

__device__ __forceinline__ void tc_free(TcSmem &sm, uint32_t ncols) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_base), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// Byte offset of element (row r, k-index k) of a panel with KC k-values in the canonical K-major
// no-swizzle layout: 8-row groups of KC/4 core matrices (8 rows x 16 bytes) each; LBO = 128 B
// (next 16-byte K chunk), SBO = KC/4 * 128 B (next 8-row group).
__device__ __forceinline__ int panel_off(int r, int k) {
    return (r >> 3) * (TC_KC / 4 * 128) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

// Round to the nearest TF32 value (10 explicit mantissa bits) in an FP32 container.
__device__ __forceinline__ float round_tf32(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// x = hi + lo with hi = rn_tf32(x) (|x - hi| <= 2^-11 |x|) and lo = rn_tf32(x - hi): both exactly
// representable in TF32, so the tensor core's TF32 read of them is exact and x - hi - lo = O(2^-22 |x|).
__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo) {
    hi = round_tf32(x);
    lo = round_tf32(x - hi);
}

// Panel staging in two halves so that global loads are batched ahead of the shared-memory stores
// (and of the MMAs of the previous panel): panel_load fetches this thread's elements of one
// (R <= 128) x KC panel of op(X) into registers (zero outside [0, nr) x [k0, K)), panel_store splits
// them into hi / lo and writes them in the canonical layout.  Element e = tid + 256 j of the panel,
// mapping t -> (row % 8, k % 4) conflict-free in shared memory; op(X)(row, k) = TX ? X[k ld + row]
// : X[row ld + k].
constexpr int TC_PER_THREAD = TC_PANEL / 256;  // elements of a 128 x KC panel per thread (blockDim 256)

__device__ __forceinline__ void panel_coords(int e, int &r, int &k) {
    const int t = e & 31, g = e >> 5;
    const int rg = g / (TC_KC / 4), kc = g % (TC_KC / 4);
    r = rg * 8 + (t & 7);
    k = kc * 4 + ((t >> 3) & 3);
}

template <bool TX>
__device__ __forceinline__ void panel_load(const float *X, int ld, int row0, int nr, int k0, int K, int R,
                                           float (&v)[TC_PER_THREAD]) {
#pragma unroll
    for (int j = 0; j < TC_PER_THREAD; ++j) {
        const int e = threadIdx.x + 256 * j;
        int r, k;
        panel_coords(e, r, k);
        v[j] = (r < R && r < nr && k0 + k < K)
                   ? __ldcg(TX ? X + (size_t)(k0 + k) * ld + row0 + r : X + (size_t)(row0 + r) * ld + k0 + k)
                   : 0.f;
    }
}

__device__ __forceinline__ void panel_store(int R, const float (&v)[TC_PER_THREAD], float *hi, float *lo) {
#pragma unroll
    for (int j = 0; j < TC_PER_THREAD; ++j) {
        const int e = threadIdx.x + 256 * j;
        int r, k;
        panel_coords(e, r, k);
        if (r < R) {
            float h, l;
            split_tf32(v[j], h, l);
            const int off = panel_off(r, k) >> 2;
            hi[off] = h;
            lo[off] = l;
        }
    }
}

// C[Mr x Nc] = (Cin ? Cin : 0) + alpha op(A)[Mr x K] op(B)[K x Nc] for the tiles t = part, part +
// nparts, ... of 128 x NT (NT = min(128, Nc rounded up to 16)); same contract as ric_gemm (Cin may
// alias C).  All threads of the CTA must call it (block size a multiple of 128).  TMEM: the
// caller allocated >= 128 columns at sm.tmem_base.
template <bool TA, bool TB>
__device__ void tc_gemm(int Mr, int Nc, int K, float alpha, const float *A, int lda, const float *Bm, int ldb,
                        const float *Cin, int ldci, float *C, int ldc, int part, int nparts, TcSmem &sm,
                        TcPhase &ph) {
    // N tile: up to 128 columns, narrower (>= 16) when a cluster would otherwise leave CTAs idle
    const int tmn = (Mr + TC_M - 1) / TC_M;
    const int want_tn = max(1, (nparts + tmn - 1) / tmn);
    const int NT = min(TC_NMAX, max(16, ((Nc + want_tn - 1) / want_tn + 15) & ~15));
    const int tnn = (Nc + NT - 1) / NT;
    const uint32_t idesc = umma_idesc_tf32(TC_M, NT);
    const int nk = (K + TC_KC - 1) / TC_KC;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int t = part; t < tmn * tnn; t += nparts) {
        const int tm = (t / tnn) * TC_M, tn = (t % tnn) * NT;
        const int nr_a = min(TC_M, Mr - tm), nr_b = min(NT, Nc - tn);
        float va[TC_PER_THREAD], vb[TC_PER_THREAD];
        panel_load<TA>(A, lda, tm, nr_a, 0, K, TC_M, va);
        panel_load<!TB>(Bm, ldb, tn, nr_b, 0, K, NT, vb);
        for (int kb = 0; kb < nk; ++kb) {
            const int buf = kb & 1;
            if (kb >= 2) {  // the MMAs that read this buffer two panels ago must be done
                mbar_wait(&sm.mbar[buf], (ph.bits >> buf) & 1u);
                ph.bits ^= 1u << buf;
            }
            panel_store(TC_M, va, sm.a_hi[buf], sm.a_lo[buf]);
            panel_store(NT, vb, sm.b_hi[buf], sm.b_lo[buf]);
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (kb + 1 < nk) {  // next panel's loads in flight while the tensor core works
                panel_load<TA>(A, lda, tm, nr_a, (kb + 1) * TC_KC, K, TC_M, va);
                panel_load<!TB>(Bm, ldb, tn, nr_b, (kb + 1) * TC_KC, K, NT, vb);
            }
            if (threadIdx.x == 0) {
                tc_fence_after();
                const uint32_t a_hi = smem_u32(sm.a_hi[buf]), a_lo = smem_u32(sm.a_lo[buf]);
                const uint32_t b_hi = smem_u32(sm.b_hi[buf]), b_lo = smem_u32(sm.b_lo[buf]);
                constexpr uint32_t LBO = 128, SBO = TC_KC / 4 * 128;
#pragma unroll
                for (int ks = 0; ks < TC_KC / 8; ++ks) {
                    const uint32_t off = ks * 256;  // two 16-byte K chunks per k-step
                    const uint32_t acc0 = (kb > 0 || ks > 0) ? 1u : 0u;
                    umma_tf32(sm.tmem_base, umma_desc(a_hi + off, LBO, SBO), umma_desc(b_hi + off, LBO, SBO), idesc, acc0);
                    umma_tf32(sm.tmem_base, umma_desc(a_hi + off, LBO, SBO), umma_desc(b_lo + off, LBO, SBO), idesc, 1u);
                    umma_tf32(sm.tmem_base, umma_desc(a_lo + off, LBO, SBO), umma_desc(b_hi + off, LBO, SBO), idesc, 1u);
                }
                umma_commit(&sm.mbar[buf]);
            }
        }
        // wait for the last panel's MMAs (and the one before it, whose barrier is still pending)
        {
            const int last = (nk - 1) & 1;
            if (nk >= 2) {
                const int other = last ^ 1;
                mbar_wait(&sm.mbar[other], (ph.bits >> other) & 1u);
                ph.bits ^= 1u << other;
            }
            mbar_wait(&sm.mbar[last], (ph.bits >> last) & 1u);
            ph.bits ^= 1u << last;
        }
        tc_fence_after();
        // epilogue: warp w reads TMEM lanes 32 (w % 4) + lane = tile rows; column chunks of 16 are
        // split between the warp quadruples
        const int quad = wid & 3, wq = wid >> 2, nq = nwarps >> 2;
        const int row = tm + quad * 32 + lane;
        for (int c0 = wq * 16; c0 < NT; c0 += 16 * nq) {
            float v[16];
            tmem_ld16(sm.tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0, v);
            if (row < Mr) {
                float cin[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {  // all Cin loads before the stores (Cin may alias C)
                    const int col = tn + c0 + j;
                    cin[j] = (Cin && col < Nc && c0 + j < NT) ? __ldcg(Cin + (size_t)row * ldci + col) : 0.f;
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int col = tn + c0 + j;
                    if (col < Nc && c0 + j < NT) C[(size_t)row * ldc + col] = fmaf(alpha, v[j], cin[j]);
                }
            }
        }
        tc_fence_before();
        __syncthreads();   // the accumulator is read before the next tile's first MMA overwrites it
        tc_fence_after();
    }
}

// Diagnostic kernel (pdilqr_debug_tc_gemm): one CTA of 256 threads computes C = Cin + op(A) op(B)
// with tc_gemm, so the descriptor / layout / 3xTF32 path can be checked in isolation.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256, 1) k_tc_gemm_test(int M, int N, int K, const float *A, int lda, const float *Bm,
                                                         int ldb, const float *Cin, float *C) {
    extern __shared__ __align__(16) unsigned char dyn[];
    TcSmem &sm = *reinterpret_cast<TcSmem *>(dyn);
    TcPhase ph;
    tc_alloc(sm, 128);
    tc_gemm<TA, TB>(M, N, K, 1.0f, A, lda, Bm, ldb, Cin, N, C, N, 0, 1, sm, ph);
    tc_free(sm, 128);
}

}  // namespace pdilqr
