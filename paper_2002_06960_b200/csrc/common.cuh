// Internal declarations shared by the librandutv.so translation units.
// All matrices are column-major FP64; i64 sizes; device pointers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <vector>

#include "../../include/randutv.h"

namespace rutv {

typedef int64_t i64;

constexpr int kNumSMs = 148;  // B200; launch heuristics only (never correctness)

// Error plumbing: kernels are launched through these so the ctx can count them
// and the first CUDA error is remembered for randutv_last_error().
void set_last_error(const char* where, cudaError_t e);
const char* last_error();

// Optional per-kernel-class timing with CUDA events on the launching stream
// (randutv_set_profiling): bench.py's roofline numbers come from here.
enum ProfKind { PK_DGEMM = 0, PK_QR_LEAF = 1, PK_JACOBI = 2, PK_GAUSSIAN = 3, PK_OTHER = 4, PK_COUNT = 5 };

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec {
    int kind;
    double flops;
    double bytes;
    size_t e0, e1;
    int64_t shape[3];  // GEMM M, N, K (for the RUTV_PROF_DUMP per-launch log)
    cudaStream_t stream;  // for the RUTV_TRACE timeline (one row per stream)
  };
  std::vector<Rec> recs;
  int64_t launches[PK_COUNT] = {0};
  double ms[PK_COUNT] = {0};
  double flops[PK_COUNT] = {0};
  double bytes[PK_COUNT] = {0};
  double busy_ms[PK_COUNT] = {0};  // union of the launch spans per kind
  size_t begin(cudaStream_t s);
  void end(cudaStream_t s, int kind, double fl, double by, size_t e0, int64_t m = 0, int64_t n = 0, int64_t k = 0);
  void collect();  // after the stream is synchronised
  void reset();
  ~Profiler();
};

struct Launch {
  cudaStream_t stream;
  int64_t* counter;  // incremented per kernel launch
  int device_sms;
  Profiler* prof = nullptr;
  // two device ints (tile counter, finished-CTA counter) private to this
  // stream: the persistent GEMM's dynamic tile scheduler (null: static tiles)
  int* sched = nullptr;
  // one CTA per GEMM tile (no persistent grid): kernels on a concurrent stream,
  // whose CTAs must retire tile by tile so other streams' kernels get SMs
  bool oneshot = false;
  // Jacobi SVD sweep cap (randutv_set_option RANDUTV_OPT_JACOBI_SWEEPS; 30 =
  // reading A10); lower it only to exercise the non-convergence status
  int jacobi_max_sweeps = 30;
  void count(int n = 1) const {
    if (counter) *counter += n;
  }
  size_t pbegin() const { return (prof && prof->on) ? prof->begin(stream) : 0; }
  void pend(int kind, double fl, double by, size_t e0, int64_t m = 0, int64_t n = 0, int64_t k = 0) const {
    if (prof && prof->on) prof->end(stream, kind, fl, by, e0, m, n, k);
  }
};

#define RUTV_CUDA(call)                                         \
  do {                                                          \
    cudaError_t e__ = (call);                                   \
    if (e__ != cudaSuccess) {                                   \
      ::rutv::set_last_error(#call, e__);                       \
      return RANDUTV_ERR_CUDA;                                  \
    }                                                           \
  } while (0)

#define RUTV_CHECK_LAUNCH(where)                                \
  do {                                                          \
    cudaError_t e__ = cudaGetLastError();                       \
    if (e__ != cudaSuccess) {                                   \
      ::rutv::set_last_error(where, e__);                       \
      return RANDUTV_ERR_CUDA;                                  \
    }                                                           \
  } while (0)

// Kernel function attributes (dynamic shared memory opt-in, cluster sizes)
// belong to a device context: `stmt` runs once per (call site, device), so a
// process driving several GPUs opts in on each; concurrent first calls may
// both run it (idempotent).  Devices >= 64 run it every time.
#define RUTV_ONCE_PER_DEVICE(stmt)                                              \
  do {                                                                          \
    static std::atomic<uint64_t> once__{0};                                     \
    int d__ = 0;                                                                \
    RUTV_CUDA(cudaGetDevice(&d__));                                             \
    const uint64_t bit__ = (d__ >= 0 && d__ < 64) ? (1ull << d__) : 0ull;       \
    if (!bit__ || !(once__.load(std::memory_order_acquire) & bit__)) {          \
      stmt;                                                                     \
      if (bit__) once__.fetch_or(bit__, std::memory_order_acq_rel);            \
    }                                                                           \
  } while (0)

// Fault injection for the error-path tests (RUTV_FAULT, read once):
//   "alloc"          the next workspace growth fails (RANDUTV_ERR_ALLOC)
//   "alloc:rank=R"   ... only on rank R of a sharded call (the pre-collective
//                    agreement must then return on every rank, none hangs)
//   "launch:N"       the N-th DGEMM launch of the process reports a CUDA
//                    error (RANDUTV_ERR_CUDA mid-factorisation)
// Tests only; unset in production.
bool fault_alloc(int rank);
bool fault_launch();

#define RUTV_TRY(expr)                                          \
  do {                                                          \
    int s__ = (expr);                                           \
    if (s__ != 0) return s__;                                   \
  } while (0)

// ---------------------------------------------------------------- launchers
// K1: G(rows x cols, ldg) of iteration `it` (philox.cu)
int launch_gaussian(const Launch& L, uint64_t seed, i64 it, i64 rows, i64 cols, double* G, i64 ldg);

// K2: C = alpha op(A) op(B) + beta C (dgemm.cu).  `ws`/`ws_elems`: split-K
// partial buffer (may be null -> no split).
int launch_dgemm(const Launch& L, bool ta, bool tb, i64 M, i64 N, i64 K, double alpha,
                 const double* A, i64 lda, const double* B, i64 ldb, double beta, double* C, i64 ldc,
                 double* ws, i64 ws_elems);
// the schedule launch_dgemm takes for the default tile configuration on `sms`
// SMs (pure host arithmetic): out = {tiles, full, tsplits, kchunk, resident, partial doubles}
int dgemm_plan(i64 M, i64 N, i64 K, i64 ws_elems, int sms, int tail_on, i64* out);

// K3/K4: panel Householder QR (qr.cu).  P (h x w, ldp) factored in place; tau (w);
// Wx: explicit unit-lower-trapezoidal W (h x w, ldw); Tf: compact-WY factor (w x w, ldtf).
struct QrWork {
  double* S;        // w x w  (W^T W)
  double* tmp1;     // w x w
  double* tmp2;     // h x w or w x (w)  trailing-update temporaries, >= h*nb and nb*w
  double* tmp3;     // nb x w
  double* partials; // leaf-kernel cross-CTA partial sums
  i64 partials_elems;
  double* gemm_ws;  // split-K buffer
  i64 gemm_ws_elems;
};
int panel_qr(const Launch& L, i64 h, i64 w, double* P, i64 ldp, double* tau, double* Wx, i64 ldw,
             double* Tf, i64 ldtf, const QrWork& qw);
i64 panel_qr_partials_elems(i64 h, i64 w);

// K7: one-sided Jacobi SVD of the w x w block B (jacobi.cu).  `status`: device
// int, set (atomicMin) to `block_id` (1-based) on non-convergence.
int launch_jacobi_svd(const Launch& L, i64 w, const double* B, i64 ldb, double* Us, double* d, double* Vs,
                      int* status, int block_id, double* scratch, i64 scratch_elems);
i64 jacobi_scratch_elems(i64 w);

// misc.cu
int launch_set_identity(const Launch& L, i64 rows, i64 cols, double* X, i64 ldx);
// X(r, c) := (r - c == shift): a shifted slice of the identity (row block of I
// for shift < 0, column panel of I for shift > 0)
int launch_set_identity_shift(const Launch& L, i64 rows, i64 cols, i64 shift, double* X, i64 ldx);
int launch_copy(const Launch& L, i64 rows, i64 cols, const double* S, i64 lds, double* D, i64 ldd);
int launch_fill(const Launch& L, i64 rows, i64 cols, double v, double* X, i64 ldx);
// zero the strictly lower part of the rows x cols block X (X = triu(X))
int launch_triu(const Launch& L, i64 rows, i64 cols, double* X, i64 ldx);
// X (w x w) := diag(d)
int launch_set_diag(const Launch& L, i64 w, const double* d, double* X, i64 ldx);
// partial sums of squares of a rows x cols block -> out[0] = ||X||_F^2 (deterministic)
int launch_sumsq(const Launch& L, i64 rows, i64 cols, const double* X, i64 ldx, double* partial, double* out);
// nonfinite scan: *flag = 1 if any NaN/Inf
int launch_nonfinite(const Launch& L, i64 rows, i64 cols, const double* X, i64 ldx, int* flag);

}  // namespace rutv
