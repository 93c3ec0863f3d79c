/*
 * include/pdilqr.h -- C ABI of libpdilqr.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of Primal-Dual iLQR (arXiv 2506.07823, "PAPER.md"; cited P:<line>).
 *
 * One call = one batched operation over B independent MPC instances, enqueued on a CUDA stream.
 * No C++ or torch types cross this boundary: plain structs, plain pointers, sizes.
 *
 * Memory ownership.  The caller owns every buffer and the workspace; the library never
 * allocates device memory and never frees caller memory.  pdilqr_create() only carves the
 * caller's workspace and copies constants.  pdilqr_linearize/solve_lq/step do no allocation and
 * no host synchronisation, so they may be captured in a CUDA graph.  The handle itself is a small
 * host object (malloc'd by create, freed by destroy).
 *
 * Layout.  Every array is dense row-major, batch-outermost, in the handle's dtype (float32 or
 * float64), 16-byte aligned, on the handle's device:
 *   A [B][N+1][n][n]   Bm[B][N+1][n][m]   c [B][N+1][n]            (dynamics, Eq. 4 / P:130-141)
 *   Q [B][N+1][n][n]   R [B][N+1][m][m]   S [B][N+1][m][n]          (Hessian blocks)
 *   q [B][N+1][n]      r [B][N+1][m]                                (gradients)
 *   P_term[B][n][n]    p_term[B][n]       dx0[B][n]                 (terminal, dx0 = xhat0 - x0)
 *   dx[B][N+2][n]  du[B][N+1][m]  dlam[B][N+2][n]  K[B][N+1][m][n]  k[B][N+1][m]
 * Stages i = 0..N carry controls; node N+1 is terminal (reading R20: N = paper's N).
 *
 * Errors.  The returned status reports argument, dimension, alignment, workspace and launch
 * errors, synchronously.  Per-instance numerical failures are reported on the device in
 * info[b] (int32): 0 = ok; k > 0 = a factorisation failed at stage k-1 (R or G not positive
 * definite, or I + C~ P~ singular in a scan combine); -1 = non-finite data, or the SRBD iterate is
 * outside the Euler-angle guard |pitch| < pi/2 - 0.1.  pdilqr_last_error() returns a message
 * for the last non-OK status of the calling thread.
 *
 * Threads / streams.  One handle per concurrent stream; handles are independent.  The device
 * is fixed at create; every call sets and restores the current device.
 */
#ifndef PDILQR_H
#define PDILQR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDILQR_ABI_VERSION 2

typedef enum {
    PDILQR_OK = 0,
    PDILQR_ERR_INVALID_ARG = 1,
    PDILQR_ERR_DIM = 2,
    PDILQR_ERR_WORKSPACE = 3,
    PDILQR_ERR_CUDA = 4,
    PDILQR_ERR_UNSUPPORTED = 5
} pdilqr_status;

typedef enum { PDILQR_F32 = 0, PDILQR_F64 = 1 } pdilqr_dtype;
typedef enum { PDILQR_MODEL_LQ = 0, PDILQR_MODEL_SRBD = 1, PDILQR_MODEL_MULTI_SRBD = 2 } pdilqr_model;

/* Built-in single-rigid-body quadruped model and its cost (SI units).
 * State x = [p(3) world, Theta(3) = ZYX (roll, pitch, yaw), v(3) world, w(3) body] (n = 12,
 * reading R13); input u = four world-frame ground reaction forces (m = 12).  Explicit Euler with
 * step dt (reading R14).  Stage cost 1/2 |x - x_ref|^2_{W_x} + 1/2 |u - u_ref|^2_{W_u} + relaxed
 * barriers on the friction pyramid and normal-force bounds of stance feet; terminal
 * cost 1/2 |x - x_ref|^2_{W_term}.  W_u = w_u_stance on stance feet, w_u_swing on swing feet. */
typedef struct {
    double dt, mass, inertia[9], gravity[3];
    double w_x[12], w_x_term[12], w_u_stance, w_u_swing;
    double mu_friction, f_min, f_max, barrier_mu, barrier_delta;
} pdilqr_srbd_params;

/* Centralized multi-robot model (PDILQR_MODEL_MULTI_SRBD; NEXT-3 of SURVEY §8(f); P:391, P:417;
 * SPEC S:449-457): n_robots copies of the SRBD model above in one OCP, n = m = 12 n_robots (state
 * and input stacked robot by robot; contact [4 R] and footholds [4 R][3] per stage likewise),
 * coupled by a collision-avoidance penalty 1/2 weight eps^2 on every robot pair at every node,
 * eps = softplus_k(d_min - d) = log(1 + exp(k (d_min - d))) / k with k = sharpness and
 * d = sqrt(|p_a - p_b|_xy^2 + 1e-6) the planar CoM distance ("a quadratic penalty term", P:391;
 * softplus smoothing), quadraticised by Gauss-Newton. */
typedef struct {
    int32_t n_robots;       /* R >= 1, 12 R <= 256                                              */
    double d_min;           /* collision distance [m] (> 0)                                     */
    double weight;          /* w >= 0                                                           */
    double sharpness;       /* k > 0                                                            */
} pdilqr_multi_params;

typedef struct {
    int32_t N;              /* horizon: stages 0..N, terminal node N+1 (N >= 0)             */
    int32_t n, m;           /* state / control dimension (SRBD: 12 / 12)                    */
    int32_t batch;          /* B, number of independent instances (>= 1)                     */
    pdilqr_dtype dtype;     /* arithmetic type of every array and of the kernels              */
    pdilqr_model model;     /* LQ: solve_lq only; SRBD: also linearize and step               */
    int32_t n_alpha;        /* line-search grid size: alpha in {2^0 .. 2^-(n_alpha-1)}; 0 -> 10 */
    double armijo_c1;       /* Armijo constant (reading R10); 0 -> 1e-4                       */
    double theta_max;       /* filter threshold on theta (reading R10); <= 0 -> 1e-2 (N+1)    */
    int32_t leaf_chunk;     /* scan leaf chunk c >= 1: elements folded sequentially per chunk,
                               chunk summaries combined by a Blelloch tree (Eq. 8).
                               1 = pure tree over all N+2 elements (n, m <= 16: Kogge-Stone /
                               Blelloch scans; 16 < n, m <= 256: Kogge-Stone levels of CTA-level
                               full combines); >= N+2 = single chunk (sequential fold).
                               0 -> library default: N+2 for batch >= 148; below that 1, except
                               for the SRBD step with batch (N+2) > 2500 (N+2 when N+2 <= 64,
                               else 8) -- the measured crossover (D1).  Large-n
                               handles take the fold unless leaf_chunk == 1.                  */
    int32_t export_policy;  /* reserved (K,k are written whenever pdilqr_dir.K/k are non-NULL) */
    pdilqr_srbd_params srbd;/* used iff model == PDILQR_MODEL_SRBD or MULTI_SRBD (per robot)  */
    pdilqr_multi_params multi; /* used iff model == PDILQR_MODEL_MULTI_SRBD                   */
} pdilqr_config;

typedef struct pdilqr_ctx *pdilqr_handle;

/* Eq. 4 data (read-only device pointers, layout above). */
typedef struct {
    const void *A, *Bm, *c, *Q, *R, *S, *q, *r, *P_term, *p_term, *dx0;
} pdilqr_lq;

/* Same layout, writable (output of pdilqr_linearize). */
typedef struct {
    void *A, *Bm, *c, *Q, *R, *S, *q, *r, *P_term, *p_term, *dx0;
} pdilqr_lq_buf;

/* Search direction (Eq. 6-7) and optional policy (Eq. 5).  K, k may be NULL. */
typedef struct {
    void *dx, *du, *dlam, *K, *k;
} pdilqr_dir;

/* SQP iterate and per-tick data of the SRBD model (device pointers).
 *   x[B][N+2][12], u[B][N+1][12], lam[B][N+2][12]  (updated in place by pdilqr_step, Eq. 16)
 *   x0[B][12] (measured state xhat0), x_ref[B][N+2][12], u_ref[B][N+1][12] or NULL (= 0),
 *   contact[B][N+1][4] uint8 (1 = stance), feet[B][N+1][4][3] world footholds. */
typedef struct {
    void *x, *u, *lam;
    const void *x0, *x_ref, *u_ref;
    const uint8_t *contact;
    const void *feet;
} pdilqr_iterate;

/* Per-instance statistics of one step (device pointers, each [B]; cost/theta/alpha in dtype):
 * cost J and constraint violation theta (Eq. 17, reading R9) at the new iterate, accepted step
 * alpha (0 if every trial was rejected), accepted flag, info code (see Errors). */
typedef struct {
    void *cost, *theta, *alpha;
    int32_t *accepted, *info;
} pdilqr_stats;

/* Bytes of device workspace a handle with this configuration needs. */
pdilqr_status pdilqr_workspace_bytes(const pdilqr_config *cfg, size_t *bytes);

/* Validate cfg, bind the caller-owned device workspace (>= pdilqr_workspace_bytes, 256-byte
 * aligned) and create a handle on CUDA device `device`.  The workspace is zero-filled once here
 * (synchronous; setup only). */
pdilqr_status pdilqr_create(const pdilqr_config *cfg, int device, void *workspace, size_t bytes,
                            pdilqr_handle *out);

pdilqr_status pdilqr_destroy(pdilqr_handle h);

/* LQ/KKT subproblem of Eq. 4 solved by the parallel associative scans of
 * element initialisation (Eq. 12-13), reverse scan with the combination rule
 * (Eq. 11, corrected as DESIGN.md readings R1-R2), per-stage policy (Eq. 5 rows),
 * forward scan of the closed-loop dynamics (Eq. 14-15, reading R6) and the dual update
 * (Eq. 7).  Writes dir->dx, du, dlam (and K, k if non-NULL); info[b] (device, may be NULL). */
pdilqr_status pdilqr_solve_lq(pdilqr_handle h, const pdilqr_lq *qp, pdilqr_dir *dir,
                              int32_t *info, void *stream /* cudaStream_t */);

/* Gradients of a scalar loss L with respect to the Eq. 4 data of pdilqr_solve_lq (same layouts
 * and dtype as pdilqr_lq; device pointers; any member may be NULL = not wanted). */
typedef struct {
    void *A, *Bm, *c, *Q, *R, *S, *q, *r, *P_term, *p_term, *dx0;
} pdilqr_lq_grad;

/* Adjoint of pdilqr_solve_lq (NEXT-4 of SURVEY §8(f): the solver made differentiable for learning,
 * P:61-62).  The LQ solution z = (dx, du, dlam) is the unique solution of the KKT
 * system M z = rhs of Eq. 4 (M symmetric: Hessian blocks Q, R, S, P_{N+1} and the constraint
 * Jacobian [A_i, B_i, -I]; rhs = -(q, r, p_{N+1}) and -(dx0, c)).  Given the upstream gradient
 * g = dL/dz (gsol: dx, du, dlam; NULL members = 0) it solves M w = g by the same parallel scans
 * (one more pdilqr_solve_lq with the handle's matrices and the linear terms q' = -g_dx[0..N],
 * r' = -g_du, p_{N+1}' = -g_dx[N+1], dx0' = -g_dlam[0], c_i' = -g_dlam[i+1]) and writes
 *   dL/dq_i = -w_dx[i], dL/dr_i = -w_du[i], dL/dp_{N+1} = -w_dx[N+1], dL/ddx0 = -w_dlam[0],
 *   dL/dc_i = -w_dlam[i+1],
 *   dL/dQ_i = -w_dx[i] dx[i]^T, dL/dR_i = -w_du[i] du[i]^T, dL/dP_{N+1} = -w_dx[N+1] dx[N+1]^T,
 *   dL/dS_i = -(w_du[i] dx[i]^T + du[i] w_dx[i]^T),
 *   dL/dA_i = -(w_dlam[i+1] dx[i]^T + dlam[i+1] w_dx[i]^T),
 *   dL/dB_i = -(w_dlam[i+1] du[i]^T + dlam[i+1] w_du[i]^T)
 * (dL = w^T (d rhs - dM z)).  The matrix gradients treat every entry as independent (symmetrise
 * for symmetric parametrisations).  sol = the forward solution of the same qp (device, required:
 * dx, du, dlam).  info as pdilqr_solve_lq.  No allocation, no host sync (graph capturable). */
pdilqr_status pdilqr_solve_lq_adjoint(pdilqr_handle h, const pdilqr_lq *qp, const pdilqr_dir *sol,
                                      const pdilqr_dir *gsol, pdilqr_lq_grad *grad, int32_t *info,
                                      void *stream);

/* SRBD linearisation + Gauss-Newton quadraticisation at the iterate (
 * q, r include the multiplier terms, reading R8).  SRBD handles only.  Exposed for inspection;
 * pdilqr_step performs it internally.  info may be NULL. */
pdilqr_status pdilqr_linearize(pdilqr_handle h, const pdilqr_iterate *it, pdilqr_lq_buf *out,
                               int32_t *info, void *stream);

/* One SQP / RTI iteration: linearise, solve the LQ subproblem by the scans, evaluate
 * the filter line search on the fixed alpha grid in parallel and apply the
 * linear update x += a dx, u += a du, lam += a dlam in place (Eq. 16).  SRBD handles only.
 * dir (may be NULL) receives the search direction. */
pdilqr_status pdilqr_step(pdilqr_handle h, pdilqr_iterate *it, pdilqr_stats *stats,
                          pdilqr_dir *dir, void *stream);

/* One closed-loop MPC tick with HOST buffers (the paper's usage): copies x0_host
 * ([B][12], dtype) into the device iterate's x0 buffer, runs pdilqr_step, and copies the first
 * control u[:,0,:] ([B][12]) and the stats back into u0_host / stats_host (host arrays of
 * [B] cost, theta, alpha in dtype followed by [B] accepted, [B] info as int32 are written to
 * the five pointers).  Host buffers should be pinned for asynchronous copies.  The call returns
 * after the copies are enqueued; synchronise the stream before reading the host outputs. */
pdilqr_status pdilqr_tick_host(pdilqr_handle h, pdilqr_iterate *it, const void *x0_host,
                               void *u0_host, void *cost_host, void *theta_host, void *alpha_host,
                               int32_t *accepted_host, int32_t *info_host, void *stream);

/* Multi-iteration solve (artifact plumbing around the one-iteration RTI of P:315;
 * SRBD handles).  Repeats pdilqr_step until every instance has converged or failed, or max_iters
 * iterations ran.  Instance b converges at iteration k when that iteration's accepted step has
 * theta <= tol and ||alpha (dx, du)||_inf <= tol, or when every alpha was rejected at a fixed
 * point: theta <= tol and |grad J . (dx, du)| <= tol max(1, |J|) (the linear model predicts no
 * decrease; R24).  A rejected step elsewhere is not convergence.  Levenberg-Marquardt
 * ladder (R28): after a factorisation failure (info > 0) or an
 * all-rejected line search away from a fixed point, the next iteration of that instance adds
 * rho = 1e-6 (then x10 per retry, up to 1e-2) to every R_i; an accepted step resets rho to 0;
 * info > 0 with rho exhausted stops the instance.  A converged instance is then frozen (later iterations neither
 * update it nor overwrite its stats with a step: they report its iterate with alpha = 0,
 * accepted = 0).  An instance whose info != 0 stops at that iteration.
 *   stats      as pdilqr_step, of each instance's last iteration (device, required)
 *   iters      device int32[B] or NULL: k > 0 converged at iteration k, -k stopped by a failure
 *              at iteration k (see stats.info), 0 = not converged within max_iters
 *   iters_run  host int32 or NULL: iterations executed (0 when max_iters = 0: iterate unchanged)
 * Host-synchronous: one 4-byte device->host read per iteration. */
pdilqr_status pdilqr_solve(pdilqr_handle h, pdilqr_iterate *it, int32_t max_iters, double tol, pdilqr_stats *stats,
                           int32_t *iters, int32_t *iters_run, void *stream);

/* Closed-loop RTI support (one SQP iteration per control tick, warm-started "with the
 * previous prediction just shifted by one time-step"; SRBD handles).
 * pdilqr_shift: x_i <- x_{i+1}, u_i <- u_{i+1}, lam_i <- lam_{i+1} in place, last entries kept.
 * The caller advances x0, x_ref, u_ref, contact and feet for the new tick. */
pdilqr_status pdilqr_shift(pdilqr_handle h, pdilqr_iterate *it, void *stream);

/* Batched SRBD plant for closed-loop simulation: integrates the handle's continuous SRBD dynamics
 * (classical RK4, `substeps` steps over dt) from x_plant[B][12] (updated in place) under the
 * zero-order-hold input u_hold[B][12] (typically u[:,0,:] of the last step), with the stage-0
 * contacts and footholds of `it` and an optional external world force ext_force[B][3] on the CoM
 * (NULL = none; e.g. the 50 N push of P:388).  Arrays in the handle's dtype, device pointers. */
pdilqr_status pdilqr_srbd_plant(pdilqr_handle h, const pdilqr_iterate *it, void *x_plant, const void *u_hold,
                                const void *ext_force, double dt, int32_t substeps, void *stream);

/* Per-kernel timing: when enabled, every kernel launch of this handle is bracketed by CUDA
 * events recorded on the launch stream (host-side bookkeeping; events are created lazily and
 * owned by the handle).  Enabling/disabling clears the records. */
pdilqr_status pdilqr_profile(pdilqr_handle h, int32_t enable);

/* Synchronises on the recorded events and aggregates them per kernel: writes up to `max`
 * entries of kernel name (static strings), launch count and total milliseconds; clears the
 * records.  Returns the number of distinct kernels (or -1 for a NULL handle). */
int32_t pdilqr_profile_read(pdilqr_handle h, int32_t max, const char **names, int32_t *launches,
                            double *total_ms);

/* Horizon sharding of one LQ problem over G ranks (NEXT-2 of SURVEY §8(f); the associative scans
 * of P:188-271 split at chunk boundaries, Eq. 8 associativity).  Rank r holds stages [s_r, e_r) of
 * the global horizon as an ordinary LQ handle (n, m <= 16; its N+1 stages, its terminal node = the
 * global node e_r).  Protocol (paper_2506_07823_b200/horizon.py):
 *   1. pdilqr_lq_segment_reduce: S_r = e_{s_r} (x) ... (x) e_{e_r - 1} (Eq. 12 elements, full rule
 *      Eq. 11 as corrected in R1/R2; in-place tree, log2 depth); all-gather S_0..S_{G-1}.
 *   2. pdilqr_lq_segment_suffix: (P, p) of S_{r+1} (x) ... (x) S_{G-1} (x) (P_term, p_term of the
 *      global problem) -- the value function at e_r; solve_lq with it as the local terminal.
 *   3. pdilqr_lq_segment_forward: F_r = (Phi, phi), the chunk's closed-loop map dx_{s_r} -> dx_{e_r}
 *      (Eq. 15 composition, R6) of Abar = A + B K, bbar = B k + c with the policy of the last
 *      solve_lq on this handle and the same qp (A, Bm, c read); all-gather F_0..F_{G-1}.
 *   4. pdilqr_lq_segment_prefix: dx_{s_r} = F_{r-1} o ... o F_0 (dx0); solve_lq with it as dx0.
 * Layouts (device, handle dtype, unpadded row-major): summary [B][3 n^2 + 2 n] = (A, C, P, b, p);
 * forward map [B][n^2 + n] = (Phi, phi); gathered arrays rank-major [G][B][...].  info (reduce) as
 * pdilqr_solve_lq.  No allocation, no host sync. */
pdilqr_status pdilqr_lq_segment_reduce(pdilqr_handle h, const pdilqr_lq *qp, void *S_out, int32_t *info, void *stream);
pdilqr_status pdilqr_lq_segment_suffix(pdilqr_handle h, const void *S_all, int32_t G, int32_t r, const void *P_term,
                                       const void *p_term, void *P_out, void *p_out, void *stream);
pdilqr_status pdilqr_lq_segment_forward(pdilqr_handle h, const pdilqr_lq *qp, void *F_out, void *stream);
pdilqr_status pdilqr_lq_segment_prefix(pdilqr_handle h, const void *F_all, int32_t G, int32_t r, const void *dx0,
                                       void *dxs_out, void *stream);

/* Diagnostic (test infrastructure for the tensor-core products of the large-n fold):
 * C[M][N] = (Cin ? Cin : 0) + op(A)[M x K] op(B)[K x N] in FP32 through the tcgen05 3xTF32 path
 * (one CTA; M, N <= 256), row-major device arrays: op(A) = A (M x K, ld lda) or A^T (A stored K x M)
 * if trans_a; same for B (K x N or N x K, ld ldb); C and Cin are M x N with ld N.  Asynchronous on
 * stream.  Returns PDILQR_ERR_DIM / INVALID_ARG / CUDA. */
pdilqr_status pdilqr_debug_tc_gemm(int32_t M, int32_t N, int32_t K, int32_t trans_a, int32_t trans_b, const float *A,
                                   int32_t lda, const float *B, int32_t ldb, const float *Cin, float *C, void *stream);

/* Number of kernels the last solve_lq / step / linearize call launched (for accounting). */
int32_t pdilqr_last_launch_count(pdilqr_handle h);

/* Thread-local message for the last non-OK status (never NULL). */
const char *pdilqr_last_error(void);

int32_t pdilqr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PDILQR_H */
