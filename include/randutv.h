/*
 * randutv.h -- C ABI of the B200-native randUTV library (librandutv.so).
 *
 * randUTV is the blocked randomized UTV factorization with power iteration of
 * Heavner, Martinsson, Quintana-Orti, "Computing rank-revealing factorizations
 * of matrices stored out-of-core" (arXiv:2002.06960), Sec. 3.1 (PAPER.md
 * P:529-688):
 *
 *     A = U T V^T,   A: m x n (m >= n),  U: m x m and V: n x n orthogonal,
 *                    T: m x n upper triangular
 *
 * built b columns at a time: per block a Gaussian G^(i), the
 * sample Y = (A_t^T A_t)^q A_t^T G, a Householder QR of Y applied
 * from the right, a Householder QR of the leading column block
 * applied from the left and an SVD of the b x b diagonal block
 * folded into U, T, V.  Conventions the paper leaves
 * open are fixed in DESIGN.md ("Readings"): Philox4x32-10 G (A7), LAPACK dlarfg
 * reflectors (A9), one-sided Jacobi SVD with tol sqrt(b)*2^-53 (A10), the final
 * block (n - k <= b) is not sampled (A5), the right transform touches all m rows
 * (A2).
 *
 * Common conventions
 *   - Every matrix is column-major FP64 (IEEE binary64) with a leading dimension
 *     ld >= rows.  Pointers are DEVICE pointers unless the function says host.
 *   - The caller owns every buffer.  The library owns only its workspace, kept
 *     in a randutv_ctx and grown on demand (one cudaMalloc per growth, never
 *     inside the factorisation loop).
 *   - All work is ordered on the ctx stream; every call synchronises that stream
 *     before returning its status.
 *   - Status codes (LAPACK "info" style):
 *        0            success
 *       -i            argument i (1-based, in the C signature) is invalid
 *       +j            the Jacobi SVD of diagonal block j (1-based, j < 2^30)
 *                     did not converge in 30 sweeps; outputs are undefined
 *       RANDUTV_ERR_* >= RANDUTV_ERR_BASE (2^30): CUDA / allocation /
 *                     non-finite-input / communicator failures
 *   - Threads: a ctx is used by one host thread at a time (its workspace,
 *     streams and events are shared by every call on it); use one ctx per
 *     thread.  The literal randutv_factor serialises its calls per device.
 *   - No CPU fallback exists: without a CUDA device every compute entry point
 *     returns RANDUTV_ERR_CUDA.
 */
#ifndef RANDUTV_H
#define RANDUTV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RANDUTV_API __attribute__((visibility("default")))

/* status codes >= RANDUTV_ERR_BASE (2^30): far above any Jacobi block index
 * +j (a factorisation has at most n / b <= 2^30 blocks), so the two never
 * collide */
#define RANDUTV_ERR_BASE      0x40000000
#define RANDUTV_ERR_CUDA      (RANDUTV_ERR_BASE + 0)  /* a CUDA runtime call failed (message: randutv_last_error) */
#define RANDUTV_ERR_ALLOC     (RANDUTV_ERR_BASE + 1)  /* device workspace allocation failed                      */
#define RANDUTV_ERR_NONFINITE (RANDUTV_ERR_BASE + 2)  /* A holds a NaN/Inf (only with RANDUTV_CHECK_FINITE)       */
#define RANDUTV_ERR_CTX       (RANDUTV_ERR_BASE + 3)  /* NULL or destroyed context                                */
#define RANDUTV_ERR_NCCL      (RANDUTV_ERR_BASE + 4)  /* NCCL missing, a collective failed or timed out           */
#define RANDUTV_ERR_NOCOMM    (RANDUTV_ERR_BASE + 5)  /* randutv_factor_dist before randutv_comm_init              */
#define RANDUTV_ERR_PEER      (RANDUTV_ERR_BASE + 6)  /* sharded call: another rank failed its argument /
                                                          workspace checks (agreed before any collective)     */

/* flags */
#define RANDUTV_NO_UV         1u    /* do not build U and V ("no orthonormal matrices") */
#define RANDUTV_CHECK_FINITE  2u    /* pre-scan A for NaN/Inf and fail with RANDUTV_ERR_NONFINITE    */
/* Re-orthonormalise the sample between power steps:
 * Y := Q(Y) before Z = A_t Y and Z := Q(Z) before Y = A_t^T Z, Q(X) the first
 * columns of X's Householder Q.  Same span as the literal products (reading
 * A8) in exact arithmetic; resolves directions below eps^(1/(2q+1)) of a
 * block's top singular value.  Costs 2q extra panel QRs per step.  Honoured by
 * randutv_factor_ex, randutv_factor_rank and randutv_factor_tol; the
 * host-streamed and sharded entries reject it (-9). */
#define RANDUTV_REORTH        4u
/* randutv_factor_ex only: enqueue the whole factorisation on the ctx stream
 * (and the ctx's side / V streams, joined back into it) and return without
 * synchronising; randutv_wait gives the status.  The call then contains no
 * host synchronisation, so after one warm-up call (which sizes the
 * workspace) it can be captured into a CUDA graph on the ctx stream and
 * replayed.  A workspace an ASYNC call has used is never freed before
 * randutv_destroy: a later call that needs more allocates a new one and the
 * old one stays valid for graphs captured over it (randutv_destroy
 * invalidates them).  Not combinable with RANDUTV_CHECK_FINITE (-9). */
#define RANDUTV_ASYNC         8u
/* randutv_factor_ex only, m > n: U is the economy m x n factor U(:, 0:n)
 * (ldu >= m), formed by backward accumulation of the left transforms
 * (reading A12) -- the paper's m x m U of a tall A is
 * often too large to hold (c4: 550 GB); A = U T(0:n, :) V^T still holds since
 * rows n..m-1 of T are zero.  Ignored for m == n.  Costs a record of the
 * reflectors (~m n doubles of workspace); not combinable with the literal
 * host-pointer entry. */
#define RANDUTV_ECON_U        16u

typedef struct randutv_ctx randutv_ctx;

/* Per-context counters, reset by randutv_reset_stats. */
typedef struct randutv_stats {
  int64_t kernel_launches;   /* kernels launched by the library on the ctx stream */
  int64_t factorizations;    /* completed randutv_factor* calls                   */
  int64_t workspace_bytes;   /* current device workspace size                     */
  int64_t h2d_bytes;         /* host->device bytes copied (host-pointer entries)  */
  int64_t d2h_bytes;         /* device->host bytes copied                          */
} randutv_stats;

/* Create a context on CUDA device `device`; `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Returns 0 or RANDUTV_ERR_*.  *ctx owns device
 * workspace only; destroy it with randutv_destroy. */
RANDUTV_API int randutv_create(randutv_ctx** ctx, int device, void* stream);
RANDUTV_API int randutv_destroy(randutv_ctx* ctx);
/* Per-ctx options.  RANDUTV_OPT_JACOBI_SWEEPS: the Jacobi SVD sweep cap, 1..30
 * (0 = the default 30 of reading A10); lowering it makes blocks fail to
 * converge, which is how the +j status path is tested.  Returns 0, -2 (unknown
 * option) or -3 (value out of range). */
#define RANDUTV_OPT_JACOBI_SWEEPS 1
/* RANDUTV_OPT_OVERSAMPLE: p >= 0 (<= 4096) extra sample columns per sampled
 * step (reading A28): G^(i) has b + p columns
 * (the first b are the draws of p = 0), Y = (A_t^T A_t)^q A_t^T G, and the b
 * directions of span(Y) along which A_t is largest are kept (Rayleigh-Ritz:
 * Q_Y, the Householder QR of A_t Q_Y and the Jacobi SVD of its R) before the
 * QR that defines V-hat.  p is capped at n - k - b per step.  0 (default) is
 * the paper's scheme.  Honoured by randutv_factor_ex / _rank / _tol; the
 * host-streamed and sharded entries return -9 while it is set. */
#define RANDUTV_OPT_OVERSAMPLE 2
RANDUTV_API int randutv_set_option(randutv_ctx* ctx, int option, int64_t value);

/* Re-bind the ctx to another stream of the same device. */
RANDUTV_API int randutv_set_stream(randutv_ctx* ctx, void* stream);

/* Device workspace (bytes) the ctx grows to for an m x n problem with block b and
 * power steps q.  Pure host arithmetic; 0 or -i. */
RANDUTV_API int randutv_workspace_bytes(int64_t m, int64_t n, int64_t b, int q, unsigned flags,
                                        size_t* bytes);

/* Literal north-star form (BASELINE.json): factor the m x n matrix A (lda >= m).
 *   U: m x m (ld m), T: m x n (ld m), V: n x n (ld n); all written.
 *   A, U, T, V are either ALL device pointers or ALL host pointers; with host
 *   pointers the call stages through device memory (whole-matrix copies on the
 *   internal stream; counted in randutv_stats.h2d/d2h_bytes).  A is read only.
 * Uses an internal context on the current CUDA device.
 * Arguments: 1 m, 2 n, 3 A, 4 lda, 5 b (block size, >= 1), 6 q (power steps,
 * >= 0), 7 seed (64-bit seed of G), 8 U, 9 T, 10 V. */
RANDUTV_API int randutv_factor(int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int q,
                               uint64_t seed, double* U, double* T, double* V);

/* Full form on device pointers.
 *   T: m x n (ldt >= m) receives the triangular factor; T may alias A exactly
 *   (T == A and ldt == lda): A is then overwritten; any other overlap is -12.
 *   U: m x m (ldu >= m), or m x n with RANDUTV_ECON_U; V: n x n (ldv >= n);
 *   both ignored (may be NULL) with RANDUTV_NO_UV.
 * Arguments: 1 ctx, 2 m, 3 n, 4 A, 5 lda, 6 b, 7 q, 8 seed, 9 flags, 10 U, 11 ldu,
 * 12 T, 13 ldt, 14 V, 15 ldv. */
RANDUTV_API int randutv_factor_ex(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                                  int64_t b, int q, uint64_t seed, unsigned flags,
                                  double* U, int64_t ldu, double* T, int64_t ldt, double* V, int64_t ldv);

/* Truncated rank-k variant: K = ceil(k/b) sampled steps, no final
 * step (if K*b >= n - b + 1 the full factorisation runs and is truncated).
 *   Uk: m x k (ldu >= m) = U(:, 0:k), formed by backward accumulation of the
 *       left transforms (reading A12), never an m x m matrix
 *   Tk: k x n (ldt >= k) = T(0:k, :)
 *   V : n x n (ldv >= n)
 *   *resid_fro (host) = ||T(k:m, k:n)||_F = ||A - Uk Tk V^T||_F
 *   *resid_2 (host, may be NULL = not computed) = ||A - Uk Tk V^T||_2 =
 *       sigma_1 of T(k:m, k:n) (SURVEY.md §8(c) reading A11): exact (QR +
 *       Jacobi SVD) when n - k <= 512; otherwise the Rayleigh-Ritz value of a
 *       512-column block Krylov space (block 32) -- a lower bound whose error
 *       decays with the gap sigma_1 / sigma_33 of the trailing block.  -1 if
 *       the small SVD did not converge.  Costs 32 pairs of skinny products
 *       with the trailing block.
 * Uk and V may be NULL with RANDUTV_NO_UV.  A is read only.
 * Arguments: 1 ctx, 2 m, 3 n, 4 A, 5 lda, 6 k, 7 b, 8 q, 9 seed, 10 flags, 11 Uk,
 * 12 ldu, 13 Tk, 14 ldt, 15 V, 16 ldv, 17 resid_fro, 18 resid_2. */
RANDUTV_API int randutv_factor_rank(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                                    int64_t k, int64_t b, int q, uint64_t seed, unsigned flags,
                                    double* Uk, int64_t ldu, double* Tk, int64_t ldt, double* V, int64_t ldv,
                                    double* resid_fro, double* resid_2);

/* Adaptive-rank variant (P:155-157 on why partial
 * methods otherwise need k up front): sampled steps run until the trailing
 * block meets ||T(k:m, k:n)||_F <= tol * ||A||_F, with k = (steps done) * b; if
 * no sampled step meets it, the full factorisation runs and k = n (rho = 0).
 * Each step adds one device-to-host norm readback.  Outputs as
 * randutv_factor_rank for that k: caller sizes Uk (ldu >= m) and Tk (ldt >= n)
 * for up to n columns / rows.  *k_out (host) receives k.
 * Arguments: 1 ctx, 2 m, 3 n, 4 A, 5 lda, 6 tol (> 0), 7 b, 8 q, 9 seed,
 * 10 flags, 11 Uk, 12 ldu, 13 Tk, 14 ldt, 15 V, 16 ldv, 17 k_out, 18 resid_fro. */
RANDUTV_API int randutv_factor_tol(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, double tol,
                                   int64_t b, int q, uint64_t seed, unsigned flags, double* Uk, int64_t ldu,
                                   double* Tk, int64_t ldt, double* V, int64_t ldv, int64_t* k_out,
                                   double* resid_fro);

/* Synchronise the ctx stream and return the status of the last RANDUTV_ASYNC
 * factorisation (0, or the 1-based block of a non-converged SVD). */
RANDUTV_API int randutv_wait(randutv_ctx* ctx);

RANDUTV_API const char* randutv_status_string(int status);
/* Last CUDA error message seen by any call of this thread ("" if none). */
RANDUTV_API const char* randutv_last_error(void);
RANDUTV_API int randutv_get_stats(randutv_ctx* ctx, randutv_stats* out);
RANDUTV_API int randutv_reset_stats(randutv_ctx* ctx);

/* Per-kernel-class timing with CUDA events recorded on the ctx stream around
 * every launch of the class (measurement support for bench.py's roofline).
 * Kinds: 0 DMMA GEMM (flops = 2MNK), 1 panel-QR leaf, 2 Jacobi SVD, 3 Gaussian,
 * 4 fold wait (time the main stream waits for the side stream's SVD + folds).
 * randutv_set_profiling(ctx, 1) resets the totals and turns recording on. */
#define RANDUTV_PROF_DGEMM    0
#define RANDUTV_PROF_QR_LEAF  1
#define RANDUTV_PROF_JACOBI   2
#define RANDUTV_PROF_GAUSSIAN 3
#define RANDUTV_PROF_FOLD_WAIT 4  /* main stream stalled on the side stream's SVD + folds */
typedef struct randutv_profile {
  int64_t launches;  /* launches recorded                                    */
  double ms;         /* summed event-to-event device time                    */
  double flops;      /* summed algorithmic flops of those launches           */
  double bytes;      /* summed compulsory bytes (operands read + C written)  */
  double busy_ms;    /* union of the launches' event spans: time during which at
                        least one launch of this kind ran (launches on the main,
                        side and V streams overlap, so busy_ms <= ms)             */
} randutv_profile;
RANDUTV_API int randutv_set_profiling(randutv_ctx* ctx, int enable);
RANDUTV_API int randutv_get_profile(randutv_ctx* ctx, int kind, randutv_profile* out);

/* ---------------------------------------------------------------------------
 * Step-level entry points (the steps S1, S2/S3, S4/S6, S8 of SURVEY.md §8(a)),
 * exported so each kernel can be parity-checked against the oracle on its own.
 * Device pointers, ctx stream, synchronous like the rest.
 * ------------------------------------------------------------------------- */

/* S1: G(0:rows, 0:cols) of iteration `it` (reading A7: Philox4x32-10,
 * counter (row>>1, col, it, 0), key (seed lo, seed hi), Box-Muller).
 * Arguments: 1 ctx, 2 seed, 3 it, 4 rows, 5 cols, 6 G, 7 ldg. */
RANDUTV_API int randutv_gaussian(randutv_ctx* ctx, uint64_t seed, int64_t it, int64_t rows, int64_t cols,
                                 double* G, int64_t ldg);

/* S2/S3/S5/S7: C := alpha op(A) op(B) + beta C with the library's FP64 DMMA
 * GEMM (op(X) = X if trans == 0, X^T if trans == 1); C is M x N.  beta == 0
 * never reads C.  Arguments: 1 ctx, 2 transa, 3 transb, 4 M, 5 N, 6 K, 7 alpha,
 * 8 A, 9 lda, 10 B, 11 ldb, 12 beta, 13 C, 14 ldc. */
RANDUTV_API int randutv_dgemm(randutv_ctx* ctx, int transa, int transb, int64_t M, int64_t N, int64_t K,
                              double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                              double beta, double* C, int64_t ldc);

/* The work schedule randutv_dgemm takes for an M x N x K product on a device
 * of `sms` SMs with a split workspace of ws_elems doubles (host arithmetic
 * only: no device, no ctx -- the time model behind split-K and the tail-split
 * of the last partial wave; S2/S3/S5/S7 all launch through it).
 * tail_split: 1 = consider splitting the last partial wave (the default path),
 * 0 = unsplit / plain split-K only.  plan (HOST, 6 int64, caller-owned):
 * [0] output tiles (64 x 64), [1] `full` = tiles computed whole over all of K,
 * [2] k-ranges per remaining tile, [3] k-range length (a multiple of 32 unless
 * unsplit), [4] resident CTA slots (3 per SM), [5] workspace doubles the
 * partial tiles occupy (<= ws_elems).  Returns 0 or -(argument index):
 * 1 M, 2 N, 3 K, 4 ws_elems, 5 sms, 6 tail_split, 7 plan. */
RANDUTV_API int randutv_dgemm_plan(int64_t M, int64_t N, int64_t K, int64_t ws_elems, int sms, int tail_split,
                                   int64_t* plan);

/* S4/S6: Householder QR of the h x w panel P (h >= w, ldp >= h) in place, LAPACK
 * dgeqrf layout (R on/above the diagonal, reflector tails below), tau (w),
 * and the compact-WY factor Tf (w x w, ldtf >= w, upper triangular, forward
 * columnwise: H_1...H_w = I - W Tf W^T).  Arguments: 1 ctx, 2 h, 3 w, 4 P, 5 ldp,
 * 6 tau, 7 Tf, 8 ldtf. */
RANDUTV_API int randutv_panel_qr(randutv_ctx* ctx, int64_t h, int64_t w, double* P, int64_t ldp,
                                 double* tau, double* Tf, int64_t ldtf);

/* S8: SVD of the w x w block B (ldb >= w, read only): B = Us diag(d) Vs^T, d >= 0
 * descending, by one-sided Jacobi (reading A10).  Us, Vs: w x w (ld w).
 * Returns +1 on non-convergence.  Arguments: 1 ctx, 2 w, 3 B, 4 ldb, 5 Us,
 * 6 d, 7 Vs. */
RANDUTV_API int randutv_small_svd(randutv_ctx* ctx, int64_t w, const double* B, int64_t ldb,
                                  double* Us, double* d, double* Vs);


/* ---------------------------------------------------------------------------
 * Host-streamed mode: the GPU analogue of the
 * paper's out-of-core randUTV, whose matrix lives on disk and moves through an
 * LRU block cache in RAM with a dedicated I/O thread overlapping transfers and
 * computation (decomposed times in Table 1).  Here
 * A, U, V live in host memory and stream as column panels (all rows x b)
 * through a device panel cache of `device_cache_bytes`, with H2D prefetch and
 * D2H write-back on two copy streams overlapping the DMMA work.
 * ------------------------------------------------------------------------- */

/* What one host-streamed factorisation moved and how long it took. */
typedef struct randutv_host_report {
  int64_t h2d_bytes;     /* host -> device panel bytes                          */
  int64_t d2h_bytes;     /* device -> host write-back bytes                     */
  int64_t cache_hits;    /* panel requests served from the device cache         */
  int64_t cache_misses;  /* panel requests that needed a (re)load               */
  int64_t cache_slots;   /* panels the cache holds                              */
  int64_t slot_bytes;    /* bytes per slot (max(m, n) * b * 8, rounded)         */
  double wall_ms;        /* device time of the whole call (events on the stream) */
  double h2d_ms;         /* summed duration of the H2D copies (I/O time)        */
  double d2h_ms;         /* summed duration of the D2H copies                   */
} randutv_host_report;

/* Full randUTV of the m x n matrix in HOST memory (A_host, lda >= m), which is
 * overwritten by T (the paper's in-place OOC factorisation); U_host (m x m,
 * ldu >= m) and V_host (n x n, ldv >= n) in host memory are written unless
 * RANDUTV_NO_UV.  Host buffers should be pinned (cudaHostAlloc /
 * torch pin_memory); unpinned ones are registered for the duration of the
 * call.  device_cache_bytes bounds the panel cache (0 = half the free device
 * memory; at least 3 panels are always used).  report (host, may be NULL)
 * receives the traffic and timing.  Results equal randutv_factor_ex's to
 * rounding (panel sums are accumulated in a different order).
 * Arguments: 1 ctx, 2 m, 3 n, 4 A_host, 5 lda, 6 b, 7 q, 8 seed, 9 flags,
 * 10 device_cache_bytes, 11 U_host, 12 ldu, 13 V_host, 14 ldv, 15 report. */
RANDUTV_API int randutv_factor_host(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b,
                                    int q, uint64_t seed, unsigned flags, size_t device_cache_bytes, double* U_host,
                                    int64_t ldu, double* V_host, int64_t ldv, randutv_host_report* report);

/* Resumable host-streamed randUTV ("resumable per
 * iteration"): runs sampled steps [step_begin, min(step_end, nsteps)) of the
 * factorisation whose state lives in the host buffers, and the final step if
 * step_end > nsteps (nsteps = ceil((n - b) / b) sampled steps).  step_begin =
 * 0 starts from A (U, V := I); step_begin = j > 0 continues from the host
 * A_host (= T after step j-1), U_host and V_host a range ending at j left
 * behind -- with the counter-based G (reading A7) the state (j, T, U, V, seed)
 * is a complete checkpoint, e.g. saved to disk between calls.  Ranges give
 * the single call's factorisation to rounding (the deferred U / V transforms
 * are merged per range).  Arguments as randutv_factor_host plus 15
 * step_begin (>= 0, <= nsteps), 16 step_end (> step_begin; INT64_MAX = to
 * the end), 17 report. */
RANDUTV_API int randutv_factor_host_steps(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda,
                                          int64_t b, int q, uint64_t seed, unsigned flags, size_t device_cache_bytes,
                                          double* U_host, int64_t ldu, double* V_host, int64_t ldv,
                                          int64_t step_begin, int64_t step_end, randutv_host_report* report);

/* ---------------------------------------------------------------------------
 * HQRRP: the paper's other factorisation, the blocked
 * randomized column-pivoted QR  A P = Q R  (Sec. 2).
 *
 * Step i (k = i b, w = min(b, n - k)): sketch Y = G^(i) R22 (b x (n-k),
 * P:330-335; G^(i) is the transpose of randUTV's Gaussian draw of (seed, i)),
 * w steps of Businger-Golub column-pivoted QR of Y pick the pivots (
 * norms recomputed each step, exact ties to the lower column), the columns
 * k:n of R (all rows) and jpvt are permuted by LAPACK dgeqp3's swap
 * convention, then the unpivoted Householder QR of the w pivoted
 * columns and its compact-WY application to the trailing columns and to Q
 * (P:372-390).  All device pointers, column-major FP64, m >= n, 1 <= b.
 *   A     (m x n, lda >= m) in: the matrix; out: R (upper trapezoidal,
 *         exact zeros below the diagonal)
 *   b     block size; min(b, n) must be <= 512 (else -6)
 *   jpvt  (n int64) out: A(:, jpvt[j]) is column j of A P (0-based)
 *   Q     (m x m, ldq >= m) out: the orthogonal factor; not touched (may be
 *         NULL) with flags & RANDUTV_NO_UV
 * Returns 0, a negative argument index (-2 m < n, -3 n, -4 A, -5 lda, -6 b,
 * -9 jpvt, -10 Q, -11 ldq) or RANDUTV_ERR_*.  Synchronous on the ctx stream.
 * ------------------------------------------------------------------------- */
RANDUTV_API int randutv_hqrrp(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t b,
                              uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq);

/* Partial HQRRP ("partial rank-revealing QR factorization"): only
 * the first K = ceil(k / b) blocks.  A is overwritten by R whose rows 0:K b
 * are final and whose trailing block R(K b:m, K b:n) is the updated,
 * unreduced remainder, so A(:, jpvt) = Q R still holds;
 * *resid_fro = ||R(k:m, k:n)||_F = ||A P - Q(:, 0:k) R(0:k, :)||_F.  Arguments
 * as randutv_hqrrp with k inserted after lda; errors are the argument
 * positions (-6 k, -7 b, -10 jpvt, -11 Q, -12 ldq).  resid_fro (host, may be
 * NULL). */
RANDUTV_API int randutv_hqrrp_rank(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t k,
                                   int64_t b, uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq,
                                   double* resid_fro);

/* HQRRP_left, host-streamed (Sec. 2.3): the left-looking HQRRP for
 * a matrix that stays in HOST memory.  Per block: the sketch Gaussian is
 * pushed through the stored reflectors (Q [0; G]), Y = (Q [0; G])^T A(:, k:n)
 * is taken over the still-unmodified remaining columns (the "repeated
 * arithmetic" of P:508-514), the CPQR of Y picks the pivots, the <= 2w host
 * columns the permutation moves are swapped, and only the current block is
 * updated (Q^* applied from the stored reflectors), factored and written back.
 *   A_host (m x n, lda >= m, host; pinned, else registered for the call)
 *          in: A; out: R on/above the diagonal and the Householder tails below
 *          it (LAPACK dgeqp3 layout: Q = H_0 H_1 ... with H_j = I - tau_j v_j v_j^T)
 *   jpvt_host (n int64, host) out: column j of A P is A(:, jpvt[j])
 *   tau_host  (n doubles, host) out: the reflector scalars
 *   report    (host, may be NULL) traffic and time (cache_slots = 2 staging slots)
 * The pivots and R equal randutv_hqrrp's up to rounding (the sketch is formed
 * in a different order).  flags must be 0 (else -8); min(b, n) <= 512.
 * Arguments: 1 ctx, 2 m, 3 n, 4 A_host, 5 lda, 6 b, 7 seed, 8 flags, 9 jpvt_host,
 * 10 tau_host, 11 report.  Synchronous. */
RANDUTV_API int randutv_hqrrp_host(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b,
                                   uint64_t seed, unsigned flags, int64_t* jpvt_host, double* tau_host,
                                   randutv_host_report* report);

/* ---------------------------------------------------------------------------
 * Multi-GPU: the column-sharded randUTV.
 *
 * The paper's method is sequential over column blocks (each sample depends on
 * the whole updated trailing matrix), but every O(r s b) product of
 * a step splits by columns.  Layout, for P ranks and block size b:
 *   A (and T): 1-D block-cyclic by column blocks of width b -- global block j
 *              (columns j*b .. min(n, (j+1)*b)) lives on rank j mod P, local
 *              blocks in increasing j; local matrix m x n_p (lda >= m);
 *   U, V     : contiguous row ranges, rows [m*p/P, m*(p+1)/P) of U (m x m) and
 *              [n*p/P, n*(p+1)/P) of V (n x n); local ld >= the row count.
 * Exchanges per sampled step: AllReduce of A_t Y (q times, (m-k) x b) and of
 * T W_V (m x b), AllGather of Y (then the same bitwise-deterministic QR(Y) on
 * every rank), Broadcast of (W_U, T_U) and of (U_s, V_s) from the owner of
 * the column block.  Results equal the single-GPU path's up to the summation
 * order of the AllReduces.
 * ------------------------------------------------------------------------- */

#define RANDUTV_UNIQUE_ID_BYTES 128

/* Pure host arithmetic (no GPU needed): the layout of rank `rank` of `nranks`.
 * out[0] = local column count n_p, out[1..2] = [first, end) row of U held,
 * out[3..4] = [first, end) row of V held.  Arguments: 1 m, 2 n, 3 b, 4 nranks,
 * 5 rank, 6 out (host, 5 int64). */
RANDUTV_API int randutv_dist_layout(int64_t m, int64_t n, int64_t b, int nranks, int rank, int64_t* out);

/* Write a fresh NCCL unique id (RANDUTV_UNIQUE_ID_BYTES bytes, host) that the
 * caller sends to every rank (e.g. torch.distributed.broadcast_object_list).
 * Returns 0 or RANDUTV_ERR_NCCL. */
RANDUTV_API int randutv_nccl_unique_id(void* out);

/* Join the NCCL communicator of `nranks` ranks (collective over all ranks; one
 * process per GPU, the ctx's device).  The ctx owns the communicator and a
 * second one split from it for the side stream; both are released by
 * randutv_destroy or a later randutv_comm_init.  Arguments: 1 ctx, 2 unique_id
 * (host, RANDUTV_UNIQUE_ID_BYTES), 3 nranks, 4 rank. */
RANDUTV_API int randutv_comm_init(randutv_ctx* ctx, const void* unique_id, int nranks, int rank);

/* Sharded full randUTV: collective over the ranks of the ctx communicator,
 * every rank passing the same m, n, b, q, seed, flags.  A_local (m x n_p,
 * device) is overwritten by the rank's columns of T.  U_local (mu x m) and
 * V_local (nv x n) receive the rank's rows of U and V (ignored with
 * RANDUTV_NO_UV).  Status: as randutv_factor_ex, identical on every rank (+j
 * Jacobi non-convergence is agreed by an AllReduce-min); RANDUTV_ERR_NOCOMM
 * without randutv_comm_init.  Before the first collective every rank's
 * argument / workspace verdict is agreed (a rank that fails returns its own
 * code, its peers RANDUTV_ERR_PEER -- nobody is left blocked in a
 * collective); waits poll ncclCommGetAsyncError and abort the communicators
 * after RUTV_NCCL_TIMEOUT_S seconds (default 1800) with RANDUTV_ERR_NCCL.
 * flags & RANDUTV_ASYNC: enqueue only (no host synchronisation, no
 * agreement: the arguments must be rank-uniform), capturable into a CUDA
 * graph with its NCCL collectives; randutv_wait gives the status.  Not with
 * RANDUTV_CHECK_FINITE or the loopback back end (-9).  Arguments: 1 ctx, 2 m, 3 n, 4 A_local, 5 lda,
 * 6 b, 7 q, 8 seed, 9 flags, 10 U_local, 11 ldu, 12 V_local, 13 ldv. */
RANDUTV_API int randutv_factor_dist(randutv_ctx* ctx, int64_t m, int64_t n, double* A_local, int64_t lda,
                                    int64_t b, int q, uint64_t seed, unsigned flags, double* U_local, int64_t ldu,
                                    double* V_local, int64_t ldv);

/* Sharded truncated rank-k randUTV (the c4 workload at 1/2/4/8
 * GPUs): K = ceil(k/b) sampled steps (k <= b * floor((n-1)/b), else -14), no
 * final step.  A_local is overwritten by the rank's columns of T (T_k = rows
 * 0:k); Uk_local (mu x k) receives rows [m*p/P, m*(p+1)/P) of U_k, formed by
 * backward accumulation of the broadcast (W_U, T_U, U_s) with one AllReduce of
 * b x (k - k_j) per step (reading A12); V_local as for randutv_factor_dist;
 * *resid_fro (host) = ||T(k:m, k:n)||_F = ||A - U_k T_k V^T||_F (identical on
 * every rank).  Invalid arguments use randutv_factor_dist's positions, plus -14
 * (k) and -15 (resid_fro).  Arguments: 1 ctx, 2 m, 3 n, 4 A_local, 5 lda, 6 k,
 * 7 b, 8 q, 9 seed, 10 flags, 11 Uk_local, 12 ldu, 13 V_local, 14 ldv,
 * 15 resid_fro. */
RANDUTV_API int randutv_factor_dist_rank(randutv_ctx* ctx, int64_t m, int64_t n, double* A_local, int64_t lda,
                                         int64_t k, int64_t b, int q, uint64_t seed, unsigned flags, double* Uk_local,
                                         int64_t ldu, double* V_local, int64_t ldv, double* resid_fro);

/* The same SPMD driver with `nranks` (<= 16) virtual ranks run as host threads
 * on ONE device, collectives done by device copies and fixed-order sums
 * between host barriers (no kernel waits on another rank).  Used to test the
 * sharded path on a single GPU.  A_locals / U_locals / V_locals: host arrays
 * of nranks device pointers laid out as for randutv_factor_dist (lda, ldu, ldv
 * shared by all ranks).  k = 0: full factorisation; k >= 1: the truncated
 * variant (U_locals hold rows of U_k, *resid_fro as randutv_factor_dist_rank).
 * Arguments: 1 device, 2 nranks, 3 m, 4 n, 5 A_locals, 6 lda, 7 b, 8 q, 9 seed,
 * 10 flags, 11 U_locals, 12 ldu, 13 V_locals, 14 ldv, 15 k, 16 resid_fro. */
RANDUTV_API int randutv_factor_dist_loopback(int device, int nranks, int64_t m, int64_t n, double* const* A_locals,
                                             int64_t lda, int64_t b, int q, uint64_t seed, unsigned flags,
                                             double* const* U_locals, int64_t ldu, double* const* V_locals,
                                             int64_t ldv, int64_t k, double* resid_fro);

/* ---------------------------------------------------------------------------
 * Sharded + host-streamed ("multi-GPU plus host
 * streaming combined"): the layout of randutv_factor_dist with every rank's
 * matrices in HOST memory, streamed through the rank's device panel cache as
 * randutv_factor_host does -- A_local_host (m x n_p, lda >= m) the rank's
 * block-cyclic columns, overwritten by T; U_local_host (mu x m, ldu >= mu)
 * and V_local_host (nv x n, ldv >= nv) its rows of U and V (row ranges of
 * randutv_dist_layout).  Per step: local sample passes with an AllReduce of Z
 * per power step, the AllGather of Y and the same QR(Y) everywhere, the T W_V
 * pass + AllReduce, the owner's panel (S5, S6, SVD), ONE broadcast of
 * [W_U | T_U | U_s | V_s], and one read-write pass over the rank's later
 * panels; U and V rows stream as in randutv_factor_host (deferred batches).
 * Results equal randutv_factor_dist's to rounding.  Collective; arguments and
 * workspace are agreed across the ranks before the first collective.  LRU
 * eviction (the Belady plan is single-GPU).  flags: RANDUTV_NO_UV only
 * (CHECK_FINITE / ASYNC / REORTH: -9).  Arguments as randutv_factor_host (the
 * sharded shapes), report (host, may be NULL) this rank's traffic. */
RANDUTV_API int randutv_factor_dist_host(randutv_ctx* ctx, int64_t m, int64_t n, double* A_local_host, int64_t lda,
                                         int64_t b, int q, uint64_t seed, unsigned flags, size_t device_cache_bytes,
                                         double* U_local_host, int64_t ldu, double* V_local_host, int64_t ldv,
                                         randutv_host_report* report);

/* randutv_factor_dist_host with `nranks` (<= 16) virtual ranks as host threads on
 * ONE device (the loopback communicator of randutv_factor_dist_loopback): the
 * single-GPU test harness.  Host pointer arrays laid out as for
 * randutv_factor_dist_host (one ld per matrix kind).  Arguments: 1 device,
 * 2 nranks, 3 m, 4 n, 5 A_locals_host, 6 lda, 7 b, 8 q, 9 seed, 10 flags,
 * 11 device_cache_bytes (per rank), 12 U_locals_host, 13 ldu, 14 V_locals_host,
 * 15 ldv. */
RANDUTV_API int randutv_factor_dist_host_loopback(int device, int nranks, int64_t m, int64_t n,
                                                  double* const* A_locals_host, int64_t lda, int64_t b, int q,
                                                  uint64_t seed, unsigned flags, size_t device_cache_bytes,
                                                  double* const* U_locals_host, int64_t ldu,
                                                  double* const* V_locals_host, int64_t ldv);

#ifdef __cplusplus
}
#endif
#endif /* RANDUTV_H */
