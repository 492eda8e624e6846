#include <algorithm>
// randUTV driver and C ABI (include/randutv.h).
//
// The host side of the hot path: one right-looking loop over column blocks of
// width b (FLAME Fig. fig:FLArandutv P:1311-1363), every
// step a handful of kernels on the ctx stream, all data resident in HBM:
//
//   sampled step i (s = n - k > b), k = i b, r = m - k, A_t = T(k:m, k:n):
//     S1  G = gaussian(seed, i)                      r x b
//     S2  Y = A_t^T G                                 s x b
//     S3  q x { Z = A_t Y ; Y = A_t^T Z }                          (A8)
//     S4  [W_V, tau_V, T_V] = QR(Y)
//     S5  T(:, k:n) -= (T(:,k:n) W_V) T_V W_V^T   (all m rows, A2)
//         V(:, k:n) -= (V(:,k:n) W_V) T_V W_V^T
//     S6  [W_U, tau_U, T_U] = QR(T(k:m, k:k+b)); keep R, zero below
//     S7  T(k:m, k+b:n) -= W_U T_U^T (W_U^T T(k:m, k+b:n))   (A3)
//         U(:, k:m) -= (U(:,k:m) W_U) T_U W_U^T
//     S8  R = U_s diag(d) V_s^T  (Jacobi)
//     S9  T11 = diag(d); T01 V_s; U_s^T T12; U1 U_s; V1 V_s
//   final step (s <= b): QR if tall, SVD of R or of the dense block, fold (A5, O10)
//   truncated: K = ceil(k/b) sampled steps, rho = ||T(k:m,k:n)||_F, U_k by
//   backward accumulation of (W_U, T_U, U_s) (A12)
//
// Workspace is carved from one cudaMalloc per ctx (grown on demand, never in
// the loop).  No CPU fallback: every arithmetic step is a kernel in this .so.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>

#include "driver.cuh"

using rutv::i64;

namespace rutv {

static thread_local char g_last_error[512] = "";

void set_last_error(const char* where, cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}
const char* last_error() { return g_last_error; }

size_t Profiler::begin(cudaStream_t s) {
  if (used == pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) {
      cudaGetLastError();
      on = false;
      return 0;
    }
    pool.push_back(e);
  }
  // inside a CUDA-graph capture a plain record only orders streams; an
  // external record becomes an event-record node that every replay re-records
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(pool[used], s, cudaEventRecordExternal);
  else
    cudaEventRecord(pool[used], s);
  return used++;
}

void Profiler::end(cudaStream_t s, int kind, double fl, double by, size_t e0, int64_t m, int64_t n, int64_t k) {
  const size_t e1 = begin(s);
  if (!on) return;
  recs.push_back(Rec{kind, fl, by, e0, e1, {m, n, k}, s});
}

void Profiler::collect() {
  // RUTV_PROF_DUMP=<file>: append one line per recorded launch (tuning only)
  static const char* dump = getenv("RUTV_PROF_DUMP");
  FILE* f = dump ? fopen(dump, "a") : nullptr;
  // spans relative to the first record's start, for the union per kind
  std::vector<std::pair<double, double>> spans[PK_COUNT];
  for (const Rec& r : recs) {
    float t = 0.f, t0 = 0.f;
    if (cudaEventElapsedTime(&t, pool[r.e0], pool[r.e1]) != cudaSuccess ||
        cudaEventElapsedTime(&t0, pool[recs[0].e0], pool[r.e0]) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    spans[r.kind].push_back({(double)t0, (double)t0 + t});
    if (f) fprintf(f, "%d %lld %lld %lld %.6f %.6e\n", r.kind, (long long)r.shape[0], (long long)r.shape[1],
                   (long long)r.shape[2], t, r.flops);
    launches[r.kind] += 1;
    ms[r.kind] += t;
    flops[r.kind] += r.flops;
    bytes[r.kind] += r.bytes;
  }
  if (f) fclose(f);
  // RUTV_TRACE=<file>: the recorded launches as a chrome://tracing / Perfetto
  // timeline, one row per stream -- the analogue of the paper's Gantt chart of
  // the task schedule (Fig. 10) without nsys
  static const char* trace = getenv("RUTV_TRACE");
  if (trace && !recs.empty()) {
    FILE* tf = fopen(trace, "w");
    if (tf) {
      static const char* names[PK_COUNT] = {"dgemm", "qr_leaf", "jacobi_svd", "gaussian", "fold_wait"};
      std::vector<cudaStream_t> ids;
      fprintf(tf, "{\"traceEvents\": [\n");
      bool first = true;
      for (const Rec& r : recs) {
        float t = 0.f, t0 = 0.f;
        if (cudaEventElapsedTime(&t, pool[r.e0], pool[r.e1]) != cudaSuccess ||
            cudaEventElapsedTime(&t0, pool[recs[0].e0], pool[r.e0]) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
        size_t sid = std::find(ids.begin(), ids.end(), r.stream) - ids.begin();
        if (sid == ids.size()) ids.push_back(r.stream);
        fprintf(tf, "%s{\"name\": \"%s %lldx%lldx%lld\", \"ph\": \"X\", \"pid\": 0, \"tid\": %zu, \"ts\": %.3f, "
                    "\"dur\": %.3f, \"args\": {\"gflop\": %.4f}}",
                first ? "" : ",\n", names[r.kind], (long long)r.shape[0], (long long)r.shape[1], (long long)r.shape[2],
                sid, 1e3 * t0, 1e3 * t, r.flops * 1e-9);
        first = false;
      }
      fprintf(tf, "\n]}\n");
      fclose(tf);
    }
  }
  for (int k = 0; k < PK_COUNT; ++k) {
    auto& v = spans[k];
    std::sort(v.begin(), v.end());
    double busy = 0.0, lo = 0.0, hi = -1.0;
    for (auto& iv : v) {
      if (iv.first > hi) {
        if (hi > lo) busy += hi - lo;
        lo = iv.first;
        hi = iv.second;
      } else if (iv.second > hi) {
        hi = iv.second;
      }
    }
    if (hi > lo) busy += hi - lo;
    busy_ms[k] += busy;
  }
  recs.clear();
  used = 0;
}

void Profiler::reset() {
  recs.clear();
  used = 0;
  for (int k = 0; k < PK_COUNT; ++k) {
    launches[k] = 0;
    ms[k] = flops[k] = bytes[k] = busy_ms[k] = 0.0;
  }
}

Profiler::~Profiler() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

}  // namespace rutv

namespace rutv {

i64 gemm_ws_elems_for(i64 m, i64 n, i64 b) {
  const i64 mx = m > n ? m : n;
  i64 e = 4 * mx * b;
  if (e < (1 << 20)) e = 1 << 20;
  return e;
}

// lefts record per step: W_U (m x b) + T_U (b x b) + U_s (b x b)
i64 lefts_elems_for(i64 m, i64 b, i64 K) { return K * (m * b + 2 * b * b); }

size_t carve(Carver& c, Work& w, i64 m, i64 n, i64 b, i64 lefts_K, bool twork) {
  const i64 mx = m > n ? m : n;
  w.G = c.take<double>(m * b);
  w.Y = c.take<double>(n * b);
  w.Z = c.take<double>(mx * b);
  w.Z2 = c.take<double>(mx * b);
  w.Zf = c.take<double>(mx * b);
  w.Acat = c.take<double>(m * 2 * b);
  w.Bt = c.take<double>(n * 2 * b);
  w.Zv = c.take<double>(mx * b);   // V stream: the V update (n rows) and the U update (m rows)
  w.Zv2 = c.take<double>(mx * b);
  w.gemm_ws_v = c.take<double>(4 * mx * b);
  w.Wv = c.take<double>(n * b);
  w.Wu = c.take<double>(m * b);
  w.TV = c.take<double>(b * b);
  w.TU = c.take<double>(b * b);
  w.Wu2 = c.take<double>(m * b);  // second (W_U, T_U) buffer of the deferred U update
  w.TU2 = c.take<double>(b * b);
  w.tauV = c.take<double>(b);
  w.tauU = c.take<double>(b);
  w.Us = c.take<double>(b * b);
  w.Vs = c.take<double>(b * b);
  w.d = c.take<double>(b);
  w.jac_elems = jacobi_scratch_elems(b);
  w.jac = c.take<double>(w.jac_elems);
  w.gemm_ws_elems = gemm_ws_elems_for(m, n, b);
  w.gemm_ws = c.take<double>(w.gemm_ws_elems);
  w.red = c.take<double>(1024);
  w.scal = c.take<double>(16);
  w.status = c.take<int>(16);
  w.flag = w.status + 4;
  w.qw.S = c.take<double>(b * b);
  w.qw.tmp1 = c.take<double>(b * 32);
  w.qw.tmp2 = c.take<double>(32 * b);
  w.qw.tmp3 = c.take<double>(32 * b);
  w.qw.partials_elems = panel_qr_partials_elems(mx, b);
  w.qw.partials = c.take<double>(w.qw.partials_elems);
  w.qw.gemm_ws = w.gemm_ws;
  w.qw.gemm_ws_elems = w.gemm_ws_elems;
  w.osR = c.take<double>(b * b);
  w.osU = c.take<double>(b * b);
  w.osV = c.take<double>(b * b);
  w.osd = c.take<double>(b);
  w.osjac = c.take<double>(jacobi_scratch_elems(b));
  w.lefts_elems = lefts_K > 0 ? lefts_elems_for(m, b, lefts_K) : 0;
  w.lefts = lefts_K > 0 ? c.take<double>(w.lefts_elems) : nullptr;
  w.Twork = twork ? c.take<double>(m * n) : nullptr;
  return c.off;
}

static const char* fault_spec() {
  static const char* f = getenv("RUTV_FAULT");
  return f ? f : "";
}

bool fault_alloc(int rank) {
  const char* f = fault_spec();
  if (strncmp(f, "alloc", 5) != 0) return false;
  const char* r = strstr(f, "rank=");
  return r ? (rank >= 0 && atoi(r + 5) == rank) : true;
}

bool fault_launch() {
  const char* f = fault_spec();
  if (strncmp(f, "launch:", 7) != 0) return false;
  static std::atomic<long> count{0};
  return ++count == atol(f + 7);
}

int ensure_ws(randutv_ctx* ctx, size_t bytes) {
  if (ctx->ws_bytes >= bytes) return 0;
  if (fault_alloc(-1)) {
    set_last_error("cudaMalloc(workspace) [RUTV_FAULT injected]", cudaErrorMemoryAllocation);
    return RANDUTV_ERR_ALLOC;
  }
  if (ctx->ws) {
    if (ctx->ws_captured) {
      // an ASYNC call (possibly captured into a CUDA graph) used it: keep it
      // alive until randutv_destroy so replays stay valid
      ctx->retired.push_back(ctx->ws);
      ctx->ws_captured = false;
    } else {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->ws);
    }
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&ctx->ws, bytes);
  if (e != cudaSuccess) {
    set_last_error("cudaMalloc(workspace)", e);
    cudaGetLastError();
    return RANDUTV_ERR_ALLOC;
  }
  ctx->ws_bytes = bytes;
  ctx->stats.workspace_bytes = (int64_t)bytes;
  return 0;
}

int prepare(randutv_ctx* ctx, Work& w, i64 m, i64 n, i64 b, i64 lefts_K, bool twork) {
  Carver dry{nullptr, 0, 0, true};
  const size_t need = carve(dry, w, m, n, b, lefts_K, twork);
  RUTV_TRY(ensure_ws(ctx, need));
  Carver real{(char*)ctx->ws, 0, ctx->ws_bytes, false};
  carve(real, w, m, n, b, lefts_K, twork);
  return 0;
}

i64 sampled_steps(i64 n, i64 b) { return n > b ? (n - b + b - 1) / b : 0; }

// ---------------------------------------------------------------- resid_2
// ||A - A_k||_2 = sigma_1 of the trailing block X = T(k:m, k:n) (r x s, r >= s;
// reading A11).  s <= kSpecM: exact -- Householder QR of a copy of X and the
// Jacobi SVD of its R.  s > kSpecM: block Krylov with Rayleigh-Ritz -- Q_0 =
// orth(Omega) (s x p, a Philox Gaussian), Y_j = X^T X Q_j, Q_{j+1} = orth(Y_j
// with Q_0..Q_j projected out twice), M = kSpecM columns in all; then
// sigma_1 ~ sqrt(lambda_max(Q^T X^T X Q)), the Gram H = Q^T [Y_0 .. Y_{J-1}]
// (M x M) by the Jacobi SVD.  The Ritz value is a lower bound that converges
// at the block-Krylov rate set by the gap sigma_1 / sigma_{p+1}.
constexpr i64 kSpecP = 32, kSpecM = 512;

struct SpecWork {
  double *Q, *Yall, *Z, *C, *H, *Us, *Vs, *d, *jac, *gemm_ws, *tau, *Wx, *Tf, *Xc;
  i64 jac_elems, gemm_ws_elems;
  QrWork qw;
  int* status;
};

size_t carve_spec(Carver& c, SpecWork& sw, i64 r, i64 s) {
  const i64 M = kSpecM, p = kSpecP;
  const bool exact = s <= M;
  const i64 w = exact ? (s > 0 ? s : 1) : M;  // Jacobi / QR width
  sw.Q = exact ? nullptr : c.take<double>(s * M);
  sw.Yall = exact ? nullptr : c.take<double>(s * M);
  sw.Z = exact ? nullptr : c.take<double>(r * p);
  sw.C = exact ? nullptr : c.take<double>(M * p);
  sw.H = c.take<double>(w * w);
  sw.Us = c.take<double>(w * w);
  sw.Vs = c.take<double>(w * w);
  sw.d = c.take<double>(w);
  sw.jac_elems = jacobi_scratch_elems(w);
  sw.jac = c.take<double>(sw.jac_elems);
  sw.gemm_ws_elems = std::max<i64>(4 * std::max(r, s) * std::max(p, exact ? w : p), 1 << 20);
  sw.gemm_ws = c.take<double>(sw.gemm_ws_elems);
  const i64 qh = exact ? r : s, qw_ = exact ? w : p;  // panels factored
  sw.tau = c.take<double>(qw_);
  sw.Wx = c.take<double>(qh * qw_);
  sw.Tf = c.take<double>(qw_ * qw_);
  sw.Xc = exact ? c.take<double>(r * w) : nullptr;
  sw.qw.S = c.take<double>(qw_ * qw_);
  sw.qw.tmp1 = c.take<double>(qw_ * 32);
  sw.qw.tmp2 = c.take<double>(32 * qw_);
  sw.qw.tmp3 = c.take<double>(32 * qw_);
  sw.qw.partials_elems = panel_qr_partials_elems(qh, qw_);
  sw.qw.partials = c.take<double>(sw.qw.partials_elems);
  sw.qw.gemm_ws = sw.gemm_ws;
  sw.qw.gemm_ws_elems = sw.gemm_ws_elems;
  sw.status = c.take<int>(4);
  return c.off;
}

// X (h x p, ld h) := the first p columns of its Householder Q (as orthonormalize)
int spec_orth(const Launch& L, SpecWork& sw, i64 h, i64 p, double* X) {
  RUTV_TRY(panel_qr(L, h, p, X, h, sw.tau, sw.Wx, h, sw.Tf, p, sw.qw));
  RUTV_TRY(launch_dgemm(L, false, true, p, p, p, 1.0, sw.Tf, p, sw.Wx, h, 0.0, sw.qw.S, p, nullptr, 0));
  RUTV_TRY(launch_set_identity(L, h, p, X, h));
  return launch_dgemm(L, false, false, h, p, p, -1.0, sw.Wx, h, sw.qw.S, p, 1.0, X, h, nullptr, 0);
}

// Enqueues the estimate; *sigma2_dev (device) receives sigma_1^2 (exact case:
// sigma_1 itself, flagged by *squared = false).
int spectral_norm(const Launch& L, SpecWork& sw, i64 r, i64 s, const double* X, i64 ldx, uint64_t seed,
                  bool* squared) {
  RUTV_CUDA(cudaMemsetAsync(sw.status, 0x7f, sizeof(int), L.stream));
  if (s <= kSpecM) {
    *squared = false;
    RUTV_TRY(launch_copy(L, r, s, X, ldx, sw.Xc, r));
    RUTV_TRY(panel_qr(L, r, s, sw.Xc, r, sw.tau, sw.Wx, r, sw.Tf, s, sw.qw));
    RUTV_TRY(launch_copy(L, s, s, sw.Xc, r, sw.H, s));
    RUTV_TRY(launch_triu(L, s, s, sw.H, s));
    return launch_jacobi_svd(L, s, sw.H, s, sw.Us, sw.d, sw.Vs, sw.status, 1, sw.jac, sw.jac_elems);
  }
  *squared = true;
  const i64 p = kSpecP, J = kSpecM / kSpecP;
  // Omega: the Philox Gaussian of a stream no factorisation step uses
  RUTV_TRY(launch_gaussian(L, seed ^ 0x5eC7A1u, 0x7fffffff, s, p, sw.Q, s));
  RUTV_TRY(spec_orth(L, sw, s, p, sw.Q));
  for (i64 j = 0; j < J; ++j) {
    double* Qj = sw.Q + j * p * s;
    double* Yj = sw.Yall + j * p * s;
    RUTV_TRY(launch_dgemm(L, false, false, r, p, s, 1.0, X, ldx, Qj, s, 0.0, sw.Z, r, sw.gemm_ws, sw.gemm_ws_elems));
    RUTV_TRY(launch_dgemm(L, true, false, s, p, r, 1.0, X, ldx, sw.Z, r, 0.0, Yj, s, sw.gemm_ws, sw.gemm_ws_elems));
    if (j + 1 == J) break;
    double* Qn = Qj + p * s;
    RUTV_TRY(launch_copy(L, s, p, Yj, s, Qn, s));
    const i64 cols = (j + 1) * p;
    for (int pass = 0; pass < 2; ++pass) {  // block classical Gram-Schmidt, twice
      RUTV_TRY(launch_dgemm(L, true, false, cols, p, s, 1.0, sw.Q, s, Qn, s, 0.0, sw.C, cols, sw.gemm_ws,
                            sw.gemm_ws_elems));
      RUTV_TRY(launch_dgemm(L, false, false, s, p, cols, -1.0, sw.Q, s, sw.C, cols, 1.0, Qn, s, nullptr, 0));
    }
    RUTV_TRY(spec_orth(L, sw, s, p, Qn));
  }
  // H = Q^T (X^T X Q), symmetrised by the Jacobi SVD's own arithmetic (PSD: d = eigenvalues)
  RUTV_TRY(launch_dgemm(L, true, false, kSpecM, kSpecM, s, 1.0, sw.Q, s, sw.Yall, s, 0.0, sw.H, kSpecM, sw.gemm_ws,
                        sw.gemm_ws_elems));
  return launch_jacobi_svd(L, kSpecM, sw.H, kSpecM, sw.Us, sw.d, sw.Vs, sw.status, 1, sw.jac, sw.jac_elems);
}

// X(rows x s, ldx) -= ((X W) Tf) W^T : the right application of Q = I - W Tf W^T
int apply_right(const Launch& L, Work& w, i64 rows, i64 s, i64 bw, double* X, i64 ldx, const double* W, i64 ldw,
                const double* Tf, i64 ldtf) {
  RUTV_TRY(launch_dgemm(L, false, false, rows, bw, s, 1.0, X, ldx, W, ldw, 0.0, w.Z, rows, w.gemm_ws,
                        w.gemm_ws_elems));
  RUTV_TRY(launch_dgemm(L, false, false, rows, bw, bw, 1.0, w.Z, rows, Tf, ldtf, 0.0, w.Z2, rows, nullptr, 0));
  RUTV_TRY(launch_dgemm(L, false, true, rows, s, bw, -1.0, w.Z2, rows, W, ldw, 1.0, X, ldx, nullptr, 0));
  return 0;
}

// X(r x c) -= W Tf^T (W^T X): the left application of Q^T
int apply_left_t(const Launch& L, Work& w, i64 r, i64 c, i64 bw, double* X, i64 ldx, const double* W, i64 ldw,
                 const double* Tf, i64 ldtf) {
  if (c <= 0) return 0;
  RUTV_TRY(launch_dgemm(L, true, false, bw, c, r, 1.0, W, ldw, X, ldx, 0.0, w.Z, bw, w.gemm_ws, w.gemm_ws_elems));
  RUTV_TRY(launch_dgemm(L, true, false, bw, c, bw, 1.0, Tf, ldtf, w.Z, bw, 0.0, w.Z2, bw, nullptr, 0));
  RUTV_TRY(launch_dgemm(L, false, false, r, c, bw, -1.0, W, ldw, w.Z2, bw, 1.0, X, ldx, nullptr, 0));
  return 0;
}

// X(rows x bw) := X M  (M bw x bw), via the temporary Zt
int right_mult_inplace(const Launch& L, double* Zt, i64 rows, i64 bw, double* X, i64 ldx, const double* M, i64 ldm) {
  if (rows <= 0) return 0;
  RUTV_TRY(launch_dgemm(L, false, false, rows, bw, bw, 1.0, X, ldx, M, ldm, 0.0, Zt, rows, nullptr, 0));
  return launch_copy(L, rows, bw, Zt, rows, X, ldx);
}

// X(bw x cols) := M^T X
int left_mult_t_inplace(const Launch& L, double* Zt, i64 bw, i64 cols, double* X, i64 ldx, const double* M, i64 ldm) {
  if (cols <= 0) return 0;
  RUTV_TRY(launch_dgemm(L, true, false, bw, cols, bw, 1.0, M, ldm, X, ldx, 0.0, Zt, bw, nullptr, 0));
  return launch_copy(L, bw, cols, Zt, bw, X, ldx);
}

// The S5 right update of the columns right of block i and the S7 left update
// as ONE rank-2b update of T (same algebra, P:1333-1336 then P:1348-1350):
// with X = T(:, cols right of block i) before S5, W2 = the rows of W_V for
// those columns and Z2 = (T W_V) T_V,
//   X'  = X - Z2 W2^T                              (S5)
//   X'' = X' - W_U T_U^T W_U^T X'(k:m)   rows k:m   (S7)
// and W_U^T X' = W_U^T X - (W_U^T Z2(k:m)) W2^T, so with
//   Y^T = (X(k:m)^T W_U - W2 (Z2(k:m)^T W_U)) T_U        (c x b)
//   X(0:k)  -= Z2(0:k) W2^T                               (K = b)
//   X(k:m)  -= [Z2(k:m) | W_U] [W2 | Y^T]^T               (K = 2b)
// one read pass (X^T W_U) and one read-modify-write pass replace the two
// read-modify-write passes and one read pass of the unfused form.
// Temporaries: w.Z (c x b), w.Bt, w.Acat.
int fused_right_left(const Launch& L, Work& w, i64 m, i64 r, i64 b, i64 kk, i64 c, double* X, i64 ldx,
                     const double* W2, i64 ldw2, const double* Z2, i64 ldz, const double* Wu, i64 ldwu,
                     const double* TU, i64 ldtu, i64 top) {
  (void)m;
  if (top < 0) top = kk;
  if (c <= 0) return 0;
  double* Ytr = w.Bt + c * b;  // second half of Bt: Y^T (c x b, ld c)
  // Pt = X(k:m)^T W_U  (c x b, K = r) -> w.Z (ld c)
  RUTV_TRY(launch_dgemm(L, true, false, c, b, r, 1.0, X + kk, ldx, Wu, ldwu, 0.0, w.Z, c, w.gemm_ws,
                        w.gemm_ws_elems));
  // Qt = Z2(k:m)^T W_U (b x b; scratch in Bt's first half), then Pt -= W2 Qt
  RUTV_TRY(launch_dgemm(L, true, false, b, b, r, 1.0, Z2 + kk, ldz, Wu, ldwu, 0.0, w.Bt, b, w.gemm_ws,
                        w.gemm_ws_elems));
  RUTV_TRY(launch_dgemm(L, false, false, c, b, b, -1.0, W2, ldw2, w.Bt, b, 1.0, w.Z, c, nullptr, 0));
  // Y^T = Pt T_U
  RUTV_TRY(launch_dgemm(L, false, false, c, b, b, 1.0, w.Z, c, TU, ldtu, 0.0, Ytr, c, nullptr, 0));
  // Bt(:, 0:b) = W2 ; Acat = [Z2(k:m) | W_U]
  RUTV_TRY(launch_copy(L, c, b, W2, ldw2, w.Bt, c));
  RUTV_TRY(launch_copy(L, r, b, Z2 + kk, ldz, w.Acat, r));
  RUTV_TRY(launch_copy(L, r, b, Wu, ldwu, w.Acat + r * b, r));
  // X(0:k) -= Z2(0:k) W2^T ; X(k:m) -= Acat Bt^T
  if (top > 0) RUTV_TRY(launch_dgemm(L, false, true, top, c, b, -1.0, Z2, ldz, W2, ldw2, 1.0, X, ldx, nullptr, 0));
  return launch_dgemm(L, false, true, r, c, 2 * b, -1.0, w.Acat, r, w.Bt, c, 1.0, X + kk, ldx, nullptr, 0);
}

// Deferring each U update to the next step's QR(Y) (Problem::udefer), with
// (W_U, T_U) double-buffered so the next column-block QR does not wait for it,
// measured c2 (n = 4096) 9.29 -> 9.53 TFLOP/s but c3 (n = 16384) 28.12 ->
// 28.03: the panel QRs are a large share of a step only for small n, so it is
// on for n <= 8192.  RUTV_UDEFER=0/1 forces it (comparison only).
bool udefer_on(i64 n) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("RUTV_UDEFER");
    v = e ? atoi(e) : -1;
  }
  return v < 0 ? n <= 8192 : v != 0;
}

// RUTV_USTREAM=0 keeps the U update on the main stream (comparison only)
bool ustream_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_USTREAM");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// RUTV_FUSE_LEFT=0 restores the separate S5 / S7 passes over T (comparison only)
bool fuse_left() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_FUSE_LEFT");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

}  // namespace rutv

namespace {

using namespace rutv;

// RUTV_VSTREAM=0 keeps the V update on the main stream (comparison only)
Launch vstream_launch(randutv_ctx* ctx) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_VSTREAM");
    v = e ? atoi(e) : 1;
  }
  if (v != 0 && fuse_left()) return ctx->v_launch();
  Launch l{nullptr, nullptr, 0, nullptr, nullptr};
  return l;
}

struct Problem {
  i64 m, n, b;
  int q;
  uint64_t seed;
  double* T;
  i64 ldt;
  double* U;  // forward m x m accumulation (may be null)
  i64 ldu;
  double* V;  // n x n (may be null)
  i64 ldv;
  bool record_lefts;
  // S8/S9 of step i run on a side stream and overlap S1-S4 of step i+1
  // (SURVEY.md §8(a) "Commutation"): eR = R and T12 of step i ready (main),
  // eF = folds of step i done (side); S5 of step i+1 waits for eF.
  Launch side;
  cudaEvent_t eR, eF;
  Launch vl;              // V stream (oneshot GEMMs); vl.stream == nullptr: V on the main stream
  cudaEvent_t eWv, eV;
  bool reorth = false;    // RANDUTV_REORTH: orthonormal Y, Z between power steps (NEXT-4)
  i64 os = 0;             // oversampling p (reading A28; randutv_set_option)
  // U update on the V stream (after the V update of the same step): it overlaps
  // the next step's sampling, S4 QR and S5; the next S6 (overwrites W_U, T_U),
  // the side stream's U fold and the final step wait for eU
  bool ustream = false;
  cudaEvent_t eWu = nullptr, eU = nullptr;
  // Deferred U update (udefer): the U update of step i is enqueued on the V
  // stream only when step i+1 reaches its QR(Y) (event eS), so it fills the
  // latency-bound panel QR of step i+1 instead of competing with the
  // GPU-saturating sampling GEMMs; eFuv = the side stream's U / V folds done
  // (eF covers only the T folds the main stream waits for)
  bool udefer = false;
  cudaEvent_t eS = nullptr, eFuv = nullptr, eUf = nullptr;
  mutable bool rec_uf = false;
  mutable bool u_pending = false;
  mutable i64 u_kk = 0, u_r = 0;
  // (W_U, T_U) double-buffered by step parity when deferring, so the next
  // column-block QR never waits for the previous U update; eUb[j]: the U
  // update reading buffer j done
  mutable int u_buf = 0;
  cudaEvent_t eUb[2] = {nullptr, nullptr};
  mutable bool rec_ub[2] = {false, false};
  mutable bool rec_fuv = false;
  // events recorded during THIS call: waits on the others are skipped (a wait
  // on an event recorded before a CUDA-graph capture began is not capturable)
  mutable bool rec_f = false, rec_v = false, rec_u = false;
  // literal host-pointer entry: column block i of T, U and V is final once the
  // folds of step i are done (later steps only touch columns >= k + b), so it
  // is copied to the (pinned) host buffers on `cps` while the next steps run
  double *hT = nullptr, *hU = nullptr, *hV = nullptr;
  cudaStream_t cps = nullptr;
  mutable i64 drained = 0;  // columns of T, U, V already copied
};

int wait_if(cudaStream_t s, cudaEvent_t e, bool recorded) {
  if (recorded) RUTV_CUDA(cudaStreamWaitEvent(s, e, 0));
  return 0;
}


// S8 + S9 for a bw x bw diagonal block at (kk, kk).  `B` is the block to
// decompose (T11 itself).
// `side`: the call runs on the side stream behind step i+1 -- the T folds are
// published by eF (the main stream waits for them), the V and U folds wait for
// the V / U updates of the step (eV, eU) and are published by eFuv
int svd_and_fold(const Launch& L, Work& w, const Problem& P, i64 kk, i64 bw, int block_id, bool side = false) {
  double* T11 = P.T + kk + kk * P.ldt;
  RUTV_TRY(launch_jacobi_svd(L, bw, T11, P.ldt, w.Us, w.d, w.Vs, w.status, block_id, w.jac, w.jac_elems));
  RUTV_TRY(launch_set_diag(L, bw, w.d, T11, P.ldt));
  RUTV_TRY(right_mult_inplace(L, w.Zf, kk, bw, P.T + kk * P.ldt, P.ldt, w.Vs, bw));                 // A01 V_s
  RUTV_TRY(left_mult_t_inplace(L, w.Zf, bw, P.n - kk - bw, P.T + kk + (kk + bw) * P.ldt, P.ldt, w.Us, bw));  // U_s^T A12
  if (side) {
    RUTV_CUDA(cudaEventRecord(P.eF, L.stream));
    P.rec_f = true;
    if (P.V && P.vl.stream) RUTV_TRY(wait_if(L.stream, P.eV, P.rec_v));
    if (P.ustream && !P.udefer) RUTV_TRY(wait_if(L.stream, P.eU, P.rec_u));
  }
  // (deferred U updates: the U fold runs on the V stream behind its U update,
  // enqueue_u_update)
  if (P.U && !(side && P.udefer))
    RUTV_TRY(right_mult_inplace(L, w.Zf, P.m, bw, P.U + kk * P.ldu, P.ldu, w.Us, bw));                // U1 U_s
  if (P.V) RUTV_TRY(right_mult_inplace(L, w.Zf, P.n, bw, P.V + kk * P.ldv, P.ldv, w.Vs, bw));         // V1 V_s
  if (side) {
    RUTV_CUDA(cudaEventRecord(P.eFuv, L.stream));
    P.rec_fuv = true;
  }
  return 0;
}

// the U update of step kk on the V stream; deferred (Problem::udefer): also
// the U fold of that step, U(:, blk) U_s, behind it -- after the side stream's
// SVD (eF) and before the next SVD overwrites U_s (eUf, waited for by the side
// stream before its next Jacobi)
int enqueue_u_update(Work& w, const Problem& P, i64 kk, i64 r, bool with_fold, int buf = 0) {
  Work wu = w;
  wu.Z = w.Zv;
  wu.Z2 = w.Zv2;
  wu.gemm_ws = w.gemm_ws_v;
  wu.gemm_ws_elems = 4 * (P.m > P.n ? P.m : P.n) * P.b;
  RUTV_TRY(apply_right(P.vl, wu, P.m, r, P.b, P.U + kk * P.ldu, P.ldu, buf ? w.Wu2 : w.Wu, r, buf ? w.TU2 : w.TU, P.b));
  if (P.udefer) {
    RUTV_CUDA(cudaEventRecord(P.eUb[buf], P.vl.stream));
    P.rec_ub[buf] = true;
  }
  if (with_fold) {
    RUTV_TRY(wait_if(P.vl.stream, P.eF, P.rec_f));
    RUTV_TRY(right_mult_inplace(P.vl, w.Zv, P.m, P.b, P.U + kk * P.ldu, P.ldu, w.Us, P.b));  // U1 U_s
    RUTV_CUDA(cudaEventRecord(P.eUf, P.vl.stream));
    P.rec_uf = true;
  }
  RUTV_CUDA(cudaEventRecord(P.eU, P.vl.stream));
  P.rec_u = true;
  return 0;
}

// a deferred U update still pending: enqueue it (and its fold) now, behind the
// main stream's progress so far
int flush_u_update(const Launch& L, Work& w, const Problem& P) {
  if (!P.u_pending) return 0;
  RUTV_CUDA(cudaEventRecord(P.eS, L.stream));
  RUTV_CUDA(cudaStreamWaitEvent(P.vl.stream, P.eS, 0));
  P.u_pending = false;
  return enqueue_u_update(w, P, P.u_kk, P.u_r, true, P.u_buf);
}

double* left_record(Work& w, const Problem& P, int step) { return w.lefts + (i64)step * (P.m * P.b + 2 * P.b * P.b); }

// (W_U, T_U) of a step for the backward U_k accumulation: on the main stream
// (the next step's S6 overwrites them there)
int record_left_w(const Launch& L, Work& w, const Problem& P, int step, i64 r, i64 bw) {
  double* rec = left_record(w, P, step);
  RUTV_TRY(launch_copy(L, r, bw, w.Wu, r, rec, r));
  return launch_copy(L, bw, bw, w.TU, P.b, rec + P.m * P.b, bw);
}

// U_s of a step: on the stream that ran its SVD
int record_left_us(const Launch& L, Work& w, const Problem& P, int step, i64 bw) {
  return launch_copy(L, bw, bw, w.Us, bw, left_record(w, P, step) + P.m * P.b + P.b * P.b, bw);
}

// RUTV_FUSE_LEFT=0 restores the separate S5 / S7 passes over T (comparison only)
bool fuse_left() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_FUSE_LEFT");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// X (h x b, ld h) := the first b columns of its Householder Q, E - W (T W_1^T)
// (oracle.randutv._orth).  Uses the S6 buffers W_U, T_U, tau_U (free until the
// column-block QR of this step) and the panel-QR scratch S for T W_1^T.
int orthonormalize(const Launch& L, Work& w, i64 h, i64 b, double* X) {
  RUTV_TRY(panel_qr(L, h, b, X, h, w.tauU, w.Wu, h, w.TU, b, w.qw));
  RUTV_TRY(launch_dgemm(L, false, true, b, b, b, 1.0, w.TU, b, w.Wu, h, 0.0, w.qw.S, b, nullptr, 0));
  RUTV_TRY(launch_set_identity(L, h, b, X, h));
  return launch_dgemm(L, false, false, h, b, b, -1.0, w.Wu, h, w.qw.S, b, 1.0, X, h, nullptr, 0);
}

// Reading A28 (oversampling; oracle.randutv._select): the
// sample Y (s x bp, bp = b + p) is reduced to the b directions of span(Y) on
// which A_t is largest -- Y := Q_Y (explicit Householder basis), B = A_t Q_Y,
// R_B from the Householder QR of B, R_B = U_R diag(d) V_R^T (Jacobi), and
// Y(:, 0:b) := Q_Y V_R(:, 0:b).  Uses the S6 buffers W_U, T_U, tau_U (the
// caller waited for the previous U update) and the os* Jacobi buffers.
int select_sample(const Launch& L, Work& w, i64 r, i64 s, i64 b, i64 bp, const double* At, i64 lda, int block_id) {
  RUTV_TRY(orthonormalize(L, w, s, bp, w.Y));
  RUTV_TRY(launch_dgemm(L, false, false, r, bp, s, 1.0, At, lda, w.Y, s, 0.0, w.Z, r, w.gemm_ws, w.gemm_ws_elems));
  RUTV_TRY(panel_qr(L, r, bp, w.Z, r, w.tauU, w.Wu, r, w.TU, bp, w.qw));
  RUTV_TRY(launch_copy(L, bp, bp, w.Z, r, w.osR, bp));
  RUTV_TRY(launch_triu(L, bp, bp, w.osR, bp));
  RUTV_TRY(launch_jacobi_svd(L, bp, w.osR, bp, w.osU, w.osd, w.osV, w.status, block_id, w.osjac,
                             jacobi_scratch_elems(bp)));
  RUTV_TRY(launch_dgemm(L, false, false, s, b, bp, 1.0, w.Y, s, w.osV, bp, 0.0, w.Z2, s, nullptr, 0));
  return launch_copy(L, s, b, w.Z2, s, w.Y, s);
}

int sampled_step(const Launch& L, Work& w, const Problem& P, i64 i) {
  const i64 m = P.m, n = P.n, b = P.b, kk = i * b, r = m - kk, s = n - kk;
  double* At = P.T + kk + kk * P.ldt;
  // oversampling: b + p sample columns, p capped at s - b (reading A28)
  const i64 pi = P.os < s - b ? P.os : s - b;
  const i64 bp = b + (pi > 0 ? pi : 0);
  // S1, S2, S3
  RUTV_TRY(launch_gaussian(L, P.seed, i, r, bp, w.G, r));
  RUTV_TRY(launch_dgemm(L, true, false, s, bp, r, 1.0, At, P.ldt, w.G, r, 0.0, w.Y, s, w.gemm_ws, w.gemm_ws_elems));
  if ((P.reorth || bp > b) && P.ustream) RUTV_TRY(wait_if(L.stream, P.eU, P.rec_u));  // W_U, T_U are reused below
  for (int qq = 0; qq < P.q; ++qq) {
    if (P.reorth) RUTV_TRY(orthonormalize(L, w, s, bp, w.Y));
    RUTV_TRY(launch_dgemm(L, false, false, r, bp, s, 1.0, At, P.ldt, w.Y, s, 0.0, w.Z, r, w.gemm_ws,
                          w.gemm_ws_elems));
    if (P.reorth) RUTV_TRY(orthonormalize(L, w, r, bp, w.Z));
    RUTV_TRY(launch_dgemm(L, true, false, s, bp, r, 1.0, At, P.ldt, w.Z, r, 0.0, w.Y, s, w.gemm_ws,
                          w.gemm_ws_elems));
  }
  if (bp > b) RUTV_TRY(select_sample(L, w, r, s, b, bp, At, P.ldt, (int)(i + 1)));
  // the previous step's deferred U update starts with this step's QR(Y)
  RUTV_TRY(flush_u_update(L, w, P));
  // S4 (overwrites W_V, T_V: the previous step's V update must have read them)
  if (P.V && P.vl.stream) RUTV_TRY(wait_if(L.stream, P.eV, P.rec_v));
  RUTV_TRY(panel_qr(L, s, b, w.Y, s, w.tauV, w.Wv, s, w.TV, b, w.qw));
  // S5 for V(:, k:n): it does not touch T, so it needs no fold event; on the V
  // stream it overlaps the QR of the column block and the T/U updates
  if (P.V) {
    if (P.vl.stream) {
      RUTV_CUDA(cudaEventRecord(P.eWv, L.stream));
      RUTV_CUDA(cudaStreamWaitEvent(P.vl.stream, P.eWv, 0));
      Work wv = w;
      wv.Z = w.Zv;
      wv.Z2 = w.Zv2;
      wv.gemm_ws = w.gemm_ws_v;
      wv.gemm_ws_elems = 4 * n * b;
      RUTV_TRY(apply_right(P.vl, wv, n, s, b, P.V + kk * P.ldv, P.ldv, w.Wv, s, w.TV, b));
      RUTV_CUDA(cudaEventRecord(P.eV, P.vl.stream));
      P.rec_v = true;
    } else {
      RUTV_TRY(apply_right(L, w, n, s, b, P.V + kk * P.ldv, P.ldv, w.Wv, s, w.TV, b));
    }
  }
  if (!fuse_left()) {
    // S5 for T: all m rows of T(:, k:n) (A2).  Row block i-1 of T(:, k:n) is
    // written by the side stream's U_s^T T12 fold of step i-1: wait for it
    // (the stall is recorded as profile kind PK_OTHER, "fold wait").
    const size_t pe = L.pbegin();
    RUTV_TRY(wait_if(L.stream, P.eF, P.rec_f));
    L.pend(PK_OTHER, 0.0, 0.0, pe);
    RUTV_TRY(apply_right(L, w, m, s, b, P.T + kk * P.ldt, P.ldt, w.Wv, s, w.TV, b));
    // S6: QR of the column block in place; keep R, zero below
    RUTV_TRY(panel_qr(L, r, b, At, P.ldt, w.tauU, w.Wu, r, w.TU, b, w.qw));
    RUTV_TRY(launch_triu(L, b, b, At, P.ldt));
    RUTV_TRY(launch_fill(L, r - b, b, 0.0, At + b, P.ldt));
    // S7
    RUTV_TRY(apply_left_t(L, w, r, s - b, b, At + b * P.ldt, P.ldt, w.Wu, r, w.TU, b));
    if (P.U) RUTV_TRY(apply_right(L, w, m, r, b, P.U + kk * P.ldu, P.ldu, w.Wu, r, w.TU, b));
  } else {
    // The side stream's folds of step i-1 write only row block i-1 of T(:, k:n)
    // (rows pk = k-b .. k, U_s^T T12), so S5-S7 of every OTHER row run before
    // waiting for them and the SVD of step i-1 hides behind the whole step:
    //   rows [0, pk) and [k, m): Z2 = (T W_V) T_V, S5 of column block i, S6 on
    //   it, the fused S5+S7 rank-2b update, the U update;
    //   then wait, and S5 of row block i-1 alone (b x s, K = b).
    const i64 pk = kk > 0 ? kk - b : 0;  // first row of the pending row block
    const i64 pb = kk - pk;              // its height (0 at step 0)
    double* Tk = P.T + kk * P.ldt;
    if (pk > 0)
      RUTV_TRY(launch_dgemm(L, false, false, pk, b, s, 1.0, Tk, P.ldt, w.Wv, s, 0.0, w.Z, m, w.gemm_ws,
                            w.gemm_ws_elems));
    RUTV_TRY(launch_dgemm(L, false, false, r, b, s, 1.0, Tk + kk, P.ldt, w.Wv, s, 0.0, w.Z + kk, m, w.gemm_ws,
                          w.gemm_ws_elems));
    if (pk > 0) RUTV_TRY(launch_dgemm(L, false, false, pk, b, b, 1.0, w.Z, m, w.TV, b, 0.0, w.Z2, m, nullptr, 0));
    RUTV_TRY(launch_dgemm(L, false, false, r, b, b, 1.0, w.Z + kk, m, w.TV, b, 0.0, w.Z2 + kk, m, nullptr, 0));
    if (pk > 0) RUTV_TRY(launch_dgemm(L, false, true, pk, b, b, -1.0, w.Z2, m, w.Wv, s, 1.0, Tk, P.ldt, nullptr, 0));
    RUTV_TRY(launch_dgemm(L, false, true, r, b, b, -1.0, w.Z2 + kk, m, w.Wv, s, 1.0, Tk + kk, P.ldt, nullptr, 0));
    const int ub = P.udefer ? (int)(i & 1) : 0;
    double* WuB = ub ? w.Wu2 : w.Wu;
    double* TUB = ub ? w.TU2 : w.TU;
    if (P.udefer) RUTV_TRY(wait_if(L.stream, P.eUb[ub], P.rec_ub[ub]));  // two steps ago: read this buffer
    else if (P.ustream) RUTV_TRY(wait_if(L.stream, P.eU, P.rec_u));     // the previous U update read W_U, T_U
    RUTV_TRY(panel_qr(L, r, b, At, P.ldt, w.tauU, WuB, r, TUB, b, w.qw));
    RUTV_TRY(launch_triu(L, b, b, At, P.ldt));
    RUTV_TRY(launch_fill(L, r - b, b, 0.0, At + b, P.ldt));
    RUTV_TRY(fused_right_left(L, w, m, r, b, kk, s - b, P.T + (kk + b) * P.ldt, P.ldt, w.Wv + b, s, w.Z2, m, WuB, r,
                              TUB, b, pk));
    if (P.U && P.ustream) {
      RUTV_CUDA(cudaEventRecord(P.eWu, L.stream));
      RUTV_CUDA(cudaStreamWaitEvent(P.vl.stream, P.eWu, 0));
      if (P.udefer) {
        P.u_pending = true;  // enqueued at the next step's QR(Y) (flush_u_update)
        P.u_kk = kk;
        P.u_r = r;
        P.u_buf = ub;
      } else {
        RUTV_TRY(enqueue_u_update(w, P, kk, r, false));
      }
    } else if (P.U) {
      RUTV_TRY(apply_right(L, w, m, r, b, P.U + kk * P.ldu, P.ldu, w.Wu, r, w.TU, b));
    }
    {
      const size_t pe = L.pbegin();
      RUTV_TRY(wait_if(L.stream, P.eF, P.rec_f));
      L.pend(PK_OTHER, 0.0, 0.0, pe);
    }
    if (pb > 0) {
      // S5 of the pending row block: T(pk:k, k:n) -= ((T(pk:k, k:n) W_V) T_V) W_V^T
      RUTV_TRY(launch_dgemm(L, false, false, pb, b, s, 1.0, Tk + pk, P.ldt, w.Wv, s, 0.0, w.Z + pk, m, w.gemm_ws,
                            w.gemm_ws_elems));
      RUTV_TRY(launch_dgemm(L, false, false, pb, b, b, 1.0, w.Z + pk, m, w.TV, b, 0.0, w.Z2 + pk, m, nullptr, 0));
      RUTV_TRY(launch_dgemm(L, false, true, pb, s, b, -1.0, w.Z2 + pk, m, w.Wv, s, 1.0, Tk + pk, P.ldt, nullptr, 0));
    }
  }
  if (P.record_lefts) RUTV_TRY(record_left_w(L, w, P, (int)i, r, b));
  // S8, S9 on the side stream, overlapping S1-S4 of step i+1
  RUTV_CUDA(cudaEventRecord(P.eR, L.stream));
  RUTV_CUDA(cudaStreamWaitEvent(P.side.stream, P.eR, 0));
  if (P.udefer) RUTV_TRY(wait_if(P.side.stream, P.eUf, P.rec_uf));  // the previous U fold read U_s
  RUTV_TRY(svd_and_fold(P.side, w, P, kk, b, (int)(i + 1), true));
  if (P.record_lefts) {
    // truncated runs: U_s recorded for the backward U_k accumulation; eFuv
    // re-recorded behind the copy (the main stream's final join waits for it)
    RUTV_TRY(record_left_us(P.side, w, P, (int)i, b));
    RUTV_CUDA(cudaEventRecord(P.eFuv, P.side.stream));
  }
  if (P.cps) {
    // block i of T, U, V is final once its U / V folds are done
    RUTV_CUDA(cudaStreamWaitEvent(P.cps, P.eFuv, 0));
    RUTV_CUDA(cudaMemcpy2DAsync(P.hT + kk * m, m * 8, P.T + kk * P.ldt, P.ldt * 8, m * 8, b, cudaMemcpyDeviceToHost,
                                P.cps));
    if (P.hU)
      RUTV_CUDA(cudaMemcpy2DAsync(P.hU + kk * m, m * 8, P.U + kk * P.ldu, P.ldu * 8, m * 8, b, cudaMemcpyDeviceToHost,
                                  P.cps));
    if (P.hV)
      RUTV_CUDA(cudaMemcpy2DAsync(P.hV + kk * n, n * 8, P.V + kk * P.ldv, P.ldv * 8, n * 8, b, cudaMemcpyDeviceToHost,
                                  P.cps));
    P.drained = kk + b;
  }
  return 0;
}

int final_step(const Launch& L, Work& w, const Problem& P, i64 i) {
  const i64 m = P.m, n = P.n, kk = i * P.b, r = m - kk, s = n - kk;
  if (s <= 0) return 0;
  double* At = P.T + kk + kk * P.ldt;
  const bool tall = r > s;
  RUTV_TRY(flush_u_update(L, w, P));
  {
    const size_t pe = L.pbegin();
    RUTV_TRY(wait_if(L.stream, P.eF, P.rec_f));  // previous step's folds
    RUTV_TRY(wait_if(L.stream, P.eFuv, P.rec_fuv));
    if (P.V && P.vl.stream) RUTV_TRY(wait_if(L.stream, P.eV, P.rec_v));
    if (P.ustream) RUTV_TRY(wait_if(L.stream, P.eU, P.rec_u));
    L.pend(PK_OTHER, 0.0, 0.0, pe);
  }
  if (tall) {
    RUTV_TRY(panel_qr(L, r, s, At, P.ldt, w.tauU, w.Wu, r, w.TU, P.b, w.qw));
    RUTV_TRY(launch_triu(L, s, s, At, P.ldt));
    RUTV_TRY(launch_fill(L, r - s, s, 0.0, At + s, P.ldt));
    if (P.U) RUTV_TRY(apply_right(L, w, m, r, s, P.U + kk * P.ldu, P.ldu, w.Wu, r, w.TU, P.b));
  }
  RUTV_TRY(svd_and_fold(L, w, P, kk, s, (int)(i + 1)));
  if (P.record_lefts) {
    if (tall) RUTV_TRY(record_left_w(L, w, P, (int)i, r, s));  // T_U has ld b in w.TU
    RUTV_TRY(record_left_us(L, w, P, (int)i, s));
  }
  return 0;
}

// Runs steps [0, nsteps) (sampled) and the final step if `with_final`; joins
// the side stream back into the main stream at the end.
int run_loop(const Launch& L, Work& w, const Problem& P, i64 nsteps, bool with_final) {
  for (i64 i = 0; i < nsteps; ++i) RUTV_TRY(sampled_step(L, w, P, i));
  if (with_final) RUTV_TRY(final_step(L, w, P, nsteps));
  RUTV_TRY(flush_u_update(L, w, P));
  RUTV_TRY(wait_if(L.stream, P.eF, P.rec_f));
  RUTV_TRY(wait_if(L.stream, P.eFuv, P.rec_fuv));
  if (P.V && P.vl.stream) RUTV_TRY(wait_if(L.stream, P.eV, P.rec_v));
  if (P.ustream) RUTV_TRY(wait_if(L.stream, P.eU, P.rec_u));
  return 0;
}

}  // namespace

namespace rutv {

int begin_call(randutv_ctx* ctx) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  RUTV_CUDA(cudaSetDevice(ctx->device));
  if (!ctx->side) {
    int lo = 0, hi = 0;
    RUTV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    RUTV_CUDA(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eR, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eF, cudaEventDisableTiming));
    RUTV_CUDA(cudaStreamCreateWithPriority(&ctx->vstr, cudaStreamNonBlocking, lo));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eWv, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eV, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eWu, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eU, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eS, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eFuv, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eUf, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eUb[0], cudaEventDisableTiming));
    RUTV_CUDA(cudaEventCreateWithFlags(&ctx->eUb[1], cudaEventDisableTiming));
  }
  return 0;
}

int finish(randutv_ctx* ctx, const Work& w) {
  int status = 0x7f7f7f7f;
  RUTV_CUDA(cudaMemcpyAsync(&status, w.status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  RUTV_CUDA(cudaGetLastError());
  if (ctx->prof.on) ctx->prof.collect();
  if (status != 0x7f7f7f7f) return status;  // 1-based block of a non-converged SVD
  return 0;
}

int start_status(randutv_ctx* ctx, const Work& w) {
  RUTV_CUDA(cudaMemsetAsync(w.status, 0x7f, sizeof(int), ctx->stream));  // 0x7f7f7f7f
  return 0;
}

int check_finite(randutv_ctx* ctx, const Launch& L, const Work& w, i64 m, i64 n, const double* A, i64 lda) {
  RUTV_CUDA(cudaMemsetAsync(w.flag, 0, sizeof(int), ctx->stream));
  RUTV_TRY(launch_nonfinite(L, m, n, A, lda, w.flag));
  int flag = 0;
  RUTV_CUDA(cudaMemcpyAsync(&flag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  return flag ? RANDUTV_ERR_NONFINITE : 0;
}

}  // namespace rutv

namespace {

using namespace rutv;

bool overlaps(const double* a, size_t abytes, const double* b, size_t bbytes) {
  const char *pa = (const char*)a, *pb = (const char*)b;
  return pa < pb + bbytes && pb < pa + abytes;
}

}  // namespace

// ============================================================================ C ABI

extern "C" {

RANDUTV_API int randutv_create(randutv_ctx** out, int device, void* stream) {
  if (!out) return -1;
  *out = nullptr;
  int ndev = 0;
  RUTV_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return -2;
  RUTV_CUDA(cudaSetDevice(device));
  int sms = 0;
  RUTV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  randutv_ctx* c = new (std::nothrow) randutv_ctx();
  if (!c) return RANDUTV_ERR_ALLOC;
  c->magic = kMagic;
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->sms = sms;
  if (cudaMalloc(&c->sched, 4 * sizeof(int)) != cudaSuccess || cudaMemset(c->sched, 0, 4 * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    c->sched = nullptr;  // static tile order
  }
  *out = c;
  return 0;
}

RANDUTV_API int randutv_destroy(randutv_ctx* ctx) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  if (ctx->ws) cudaFree(ctx->ws);
  for (void* p : ctx->retired) cudaFree(p);
  ctx->retired.clear();
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->sched) cudaFree(ctx->sched);
  rutv::comm_free(ctx->comm_side);
  rutv::comm_free(ctx->comm);
  ctx->comm = ctx->comm_side = nullptr;
  if (ctx->vstr) {
    cudaStreamSynchronize(ctx->vstr);
    cudaEventDestroy(ctx->eWv);
    cudaEventDestroy(ctx->eV);
    cudaEventDestroy(ctx->eWu);
    cudaEventDestroy(ctx->eU);
    cudaEventDestroy(ctx->eS);
    cudaEventDestroy(ctx->eFuv);
    cudaEventDestroy(ctx->eUf);
    cudaEventDestroy(ctx->eUb[0]);
    cudaEventDestroy(ctx->eUb[1]);
    cudaStreamDestroy(ctx->vstr);
  }
  if (ctx->cps) {
    cudaStreamSynchronize(ctx->cps);
    cudaStreamDestroy(ctx->cps);
  }
  if (ctx->cstr) {
    cudaStreamSynchronize(ctx->cstr);
    for (cudaEvent_t e : ctx->ecomm) cudaEventDestroy(e);
    cudaStreamDestroy(ctx->cstr);
  }
  if (ctx->side) {
    cudaEventDestroy(ctx->eR);
    cudaEventDestroy(ctx->eF);
    cudaStreamDestroy(ctx->side);
  }
  ctx->magic = 0;
  delete ctx;
  return 0;
}

RANDUTV_API int randutv_set_option(randutv_ctx* ctx, int option, int64_t value) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  if (option == RANDUTV_OPT_JACOBI_SWEEPS) {
    if (value < 0 || value > 30) return -3;
    ctx->jacobi_max_sweeps = (int)value;
    return 0;
  }
  if (option == RANDUTV_OPT_OVERSAMPLE) {
    if (value < 0 || value > 4096) return -3;
    ctx->oversample = value;
    return 0;
  }
  return -2;
}

RANDUTV_API int randutv_set_stream(randutv_ctx* ctx, void* stream) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  ctx->stream = (cudaStream_t)stream;
  return 0;
}

RANDUTV_API int randutv_get_stats(randutv_ctx* ctx, randutv_stats* out) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  if (!out) return -2;
  *out = ctx->stats;
  return 0;
}

RANDUTV_API int randutv_reset_stats(randutv_ctx* ctx) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  const int64_t ws = ctx->stats.workspace_bytes;
  memset(&ctx->stats, 0, sizeof(ctx->stats));
  ctx->stats.workspace_bytes = ws;
  return 0;
}

RANDUTV_API const char* randutv_last_error(void) { return rutv::last_error(); }

RANDUTV_API int randutv_set_profiling(randutv_ctx* ctx, int enable) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  ctx->prof.reset();
  ctx->prof.on = enable != 0;
  return 0;
}

RANDUTV_API int randutv_get_profile(randutv_ctx* ctx, int kind, randutv_profile* out) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  if (kind < 0 || kind >= rutv::PK_COUNT) return -2;
  if (!out) return -3;
  out->launches = ctx->prof.launches[kind];
  out->ms = ctx->prof.ms[kind];
  out->flops = ctx->prof.flops[kind];
  out->bytes = ctx->prof.bytes[kind];
  out->busy_ms = ctx->prof.busy_ms[kind];
  return 0;
}

RANDUTV_API const char* randutv_status_string(int s) {
  if (s == 0) return "success";
  if (s < 0) return "invalid argument (see the 1-based index in the status)";
  if (s == RANDUTV_ERR_CUDA) return "CUDA runtime error (randutv_last_error has the message)";
  if (s == RANDUTV_ERR_ALLOC) return "device workspace allocation failed";
  if (s == RANDUTV_ERR_NONFINITE) return "input matrix holds NaN or Inf";
  if (s == RANDUTV_ERR_CTX) return "invalid or destroyed context";
  if (s == RANDUTV_ERR_NCCL) return "NCCL missing, or a collective failed or timed out (randutv_last_error)";
  if (s == RANDUTV_ERR_NOCOMM) return "sharded entry called before randutv_comm_init";
  if (s == RANDUTV_ERR_PEER) return "another rank of the sharded call rejected its arguments or workspace";
  if (s >= RANDUTV_ERR_BASE) return "unknown error";
  return "Jacobi SVD of a diagonal block did not converge (status = 1-based block index)";
}

RANDUTV_API int randutv_workspace_bytes(int64_t m, int64_t n, int64_t b, int q, unsigned flags, size_t* bytes) {
  if (m < n) return -1;
  if (n < 1) return -2;
  if (b < 1) return -3;
  if (q < 0) return -4;
  if (!bytes) return -6;
  (void)flags;
  const i64 bb = b < n ? b : n;
  Work w;
  Carver dry{nullptr, 0, 0, true};
  *bytes = carve(dry, w, m, n, bb, 0, false);
  return 0;
}

namespace {
int backward_uk(const rutv::Launch& L, rutv::Work& w, rutv::i64 m, rutv::i64 n, rutv::i64 bb, rutv::i64 nrec,
                bool with_final, rutv::i64 k, double* Uk, rutv::i64 ldu);
}

struct Drain {
  double *hT, *hU, *hV;  // pinned host T (m x n), U (m x m), V (n x n), ld = rows
  i64 drained;           // out: columns already copied
};

static int factor_ex_impl(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int q,
                          uint64_t seed, unsigned flags, double* U, int64_t ldu, double* T, int64_t ldt, double* V,
                          int64_t ldv, Drain* dr);

// A call that fails after enqueuing work must not return while that work can
// still write the caller's buffers (the side / V / copy streams included)
static int drain_on_error(randutv_ctx* ctx, int st) {
  if (st == 0 || (st > 0 && st < RANDUTV_ERR_BASE) || !ctx || ctx->magic != rutv::kMagic) return st;
  for (cudaStream_t s : {ctx->stream, ctx->side, ctx->vstr, ctx->cps})
    if (s) cudaStreamSynchronize(s);
  cudaGetLastError();
  return st;
}

RANDUTV_API int randutv_factor_ex(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b,
                                  int q, uint64_t seed, unsigned flags, double* U, int64_t ldu, double* T,
                                  int64_t ldt, double* V, int64_t ldv) {
  return drain_on_error(ctx, factor_ex_impl(ctx, m, n, A, lda, b, q, seed, flags, U, ldu, T, ldt, V, ldv, nullptr));
}

static int factor_ex_impl(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int q,
                          uint64_t seed, unsigned flags, double* U, int64_t ldu, double* T, int64_t ldt, double* V,
                          int64_t ldv, Drain* dr) {
  RUTV_TRY(begin_call(ctx));
  const bool uv = !(flags & RANDUTV_NO_UV);
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A) return -4;
  if (lda < m) return -5;
  if (b < 1) return -6;
  if (q < 0) return -7;
  if (uv && !U) return -10;
  if (uv && ldu < m) return -11;
  if (!T) return -12;
  if (ldt < m) return -13;
  if (uv && !V) return -14;
  if (uv && ldv < n) return -15;
  if ((flags & RANDUTV_ASYNC) && (flags & RANDUTV_CHECK_FINITE)) return -9;  // the scan synchronises
  // economy U (m x n) by backward accumulation (reading A12); for m == n it is
  // the full U and the forward accumulation is kept
  const bool econ = uv && (flags & RANDUTV_ECON_U) && m > n;
  if (econ && dr) return -9;
  const bool alias = (T == A);
  if (alias && ldt != lda) return -13;
  if (!alias && overlaps(A, (size_t)lda * n * 8, T, (size_t)ldt * n * 8)) return -12;
  const i64 bb = b < n ? b : n;
  const i64 nsamp = sampled_steps(n, bb);
  const i64 nrec = econ ? nsamp + 1 : 0;
  Launch L = ctx->launch();
  Work w;
  RUTV_TRY(prepare(ctx, w, m, n, bb + ctx->oversample, nrec, false));
  if (flags & RANDUTV_CHECK_FINITE) RUTV_TRY(check_finite(ctx, L, w, m, n, A, lda));
  RUTV_TRY(start_status(ctx, w));
  if (!alias) RUTV_CUDA(cudaMemcpy2DAsync(T, ldt * 8, A, lda * 8, m * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (uv) {
    if (!econ) RUTV_TRY(launch_set_identity(L, m, m, U, ldu));
    RUTV_TRY(launch_set_identity(L, n, n, V, ldv));
  }
  Problem P{m, n, bb, q, seed, T, ldt, (uv && !econ) ? U : nullptr, ldu, uv ? V : nullptr, ldv, econ,
            ctx->side_launch(), ctx->eR, ctx->eF, vstream_launch(ctx), ctx->eWv, ctx->eV};
  P.reorth = (flags & RANDUTV_REORTH) != 0;
  P.os = ctx->oversample;
  P.ustream = P.U && P.vl.stream && ustream_on();
  P.eWu = ctx->eWu;
  P.eU = ctx->eU;
  P.eS = ctx->eS;
  P.eFuv = ctx->eFuv;
  P.eUf = ctx->eUf;
  P.eUb[0] = ctx->eUb[0];
  P.eUb[1] = ctx->eUb[1];
  // deferral needs W_U, T_U intact until the next QR(Y): the re-orthonormalised
  // and oversampled power steps reuse them before it; the literal entry's
  // column-block drain needs each block final at the end of its step
  P.udefer = P.ustream && udefer_on(n) && !P.reorth && ctx->oversample == 0 && !dr;
  if (dr && uv) {
    if (!ctx->cps) RUTV_CUDA(cudaStreamCreateWithFlags(&ctx->cps, cudaStreamNonBlocking));
    P.cps = ctx->cps;
    P.hT = dr->hT;
    P.hU = dr->hU;
    P.hV = dr->hV;
  }
  RUTV_TRY(run_loop(L, w, P, nsamp, true));
  if (econ) RUTV_TRY(backward_uk(L, w, m, n, bb, nrec, true, n, U, ldu));
  if (P.cps) {
    // the main stream (and so finish) waits for the drained copies too
    RUTV_CUDA(cudaEventRecord(ctx->eWu, P.cps));
    RUTV_CUDA(cudaStreamWaitEvent(L.stream, ctx->eWu, 0));
    dr->drained = P.drained;
  }
  if (flags & RANDUTV_ASYNC) {
    // enqueued only: the status word stays on the device (randutv_wait)
    ctx->async_status = w.status;
    ctx->async_dist = false;
    ctx->ws_captured = true;
    ctx->stats.factorizations++;
    return 0;
  }
  const int st = finish(ctx, w);
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

RANDUTV_API int randutv_wait(randutv_ctx* ctx) {
  if (!ctx || ctx->magic != kMagic) return RANDUTV_ERR_CTX;
  RUTV_CUDA(cudaSetDevice(ctx->device));
  if (ctx->async_dist && ctx->comm) RUTV_TRY(rutv::comm_sync(ctx->comm, ctx->stream));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  // per-kernel events of the async call (or of the last replay of a graph
  // captured with profiling on)
  if (ctx->prof.on) ctx->prof.collect();
  if (!ctx->async_status) return 0;
  int status = 0x7f7f7f7f;
  RUTV_CUDA(cudaMemcpy(&status, ctx->async_status, sizeof(int), cudaMemcpyDeviceToHost));
  return status == 0x7f7f7f7f ? 0 : status;
}

}  // extern "C"

namespace {

// U_k = U^(1) ... U^(p) [I_k; 0] = U(:, 0:k) by backward accumulation of the
// recorded left transforms (reading A12): X := [I_k; 0]; for j = nrec-1 .. 0:
// X(k_j:k_j+w_j, :) := U_s^(j) X(...); X(k_j:m, :) -= W_j (T_j (W_j^T X(k_j:m, :))).
// The last record is the final step's when `with_final` (width n - k_j; no
// reflectors if that block was square).
int backward_uk(const Launch& L, Work& w, i64 m, i64 n, i64 bb, i64 nrec, bool with_final, i64 k, double* Uk,
                i64 ldu) {
  RUTV_TRY(launch_set_identity(L, m, k, Uk, ldu));
  for (i64 j = nrec - 1; j >= 0; --j) {
    const i64 kj = j * bb;
    if (kj >= k) continue;
    const bool fin = with_final && j == nrec - 1;
    const i64 wj = fin ? n - kj : bb;
    const i64 rj = m - kj;
    const bool has_w = !fin || rj > wj;
    const double* rec = w.lefts + j * (m * bb + 2 * bb * bb);
    const i64 cols = k - kj;
    double* X = Uk + kj + kj * ldu;  // rows kj.., cols kj..k
    // X(0:wj, :) = U_s X(0:wj, :)
    RUTV_TRY(launch_dgemm(L, false, false, wj, cols, wj, 1.0, rec + m * bb + bb * bb, wj, X, ldu, 0.0, w.Z, wj,
                          nullptr, 0));
    RUTV_TRY(launch_copy(L, wj, cols, w.Z, wj, X, ldu));
    if (has_w) {
      // X(kj:m) -= W (T (W^T X))
      RUTV_TRY(launch_dgemm(L, true, false, wj, cols, rj, 1.0, rec, rj, X, ldu, 0.0, w.Z, wj, w.gemm_ws,
                            w.gemm_ws_elems));
      RUTV_TRY(launch_dgemm(L, false, false, wj, cols, wj, 1.0, rec + m * bb, wj, w.Z, wj, 0.0, w.Z2, wj, nullptr,
                            0));
      RUTV_TRY(launch_dgemm(L, false, false, rj, cols, wj, -1.0, rec, rj, w.Z2, wj, 1.0, X, ldu, nullptr, 0));
    }
  }
  return 0;
}

// The truncated variant (fixed k) and the adaptive-rank variant (tol > 0: stop
// after the first sampled step whose trailing block has ||T(k:m,k:n)||_F <=
// tol ||A||_F; P:155-157 on why partial methods
// otherwise need k up front).  Status, outputs and argument positions follow
// randutv_factor_rank; *k_out receives the rank used.
int truncated_impl(randutv_ctx* ctx, i64 m, i64 n, const double* A, i64 lda, i64 k, double tol, i64 b, int q,
                   uint64_t seed, unsigned flags, double* Uk, i64 ldu, double* Tk, i64 ldt, double* V, i64 ldv,
                   double* resid_fro, int64_t* k_out, double* resid_2 = nullptr) {
  const bool adaptive = tol > 0.0;
  const bool uv = !(flags & RANDUTV_NO_UV);
  const i64 bb = b < n ? b : n;
  const i64 nsamp = sampled_steps(n, bb);
  i64 K = adaptive ? nsamp : (k + bb - 1) / bb;
  bool with_final = adaptive;  // adaptive: the full factorisation if no step meets tol
  if (!adaptive && K > nsamp) {
    K = nsamp;
    with_final = true;
  }
  const i64 nrec_max = uv ? K + (with_final ? 1 : 0) : 0;
  Launch L = ctx->launch();
  Work w;
  SpecWork sw{};
  if (resid_2) {
    // the main workspace followed by the resid_2 region (fixed k: the
    // trailing block is (m - k) x (n - k))
    Carver dry{nullptr, 0, 0, true};
    carve(dry, w, m, n, bb + ctx->oversample, nrec_max, true);
    carve_spec(dry, sw, m - k, n - k);
    RUTV_TRY(ensure_ws(ctx, dry.off));
    Carver real{(char*)ctx->ws, 0, ctx->ws_bytes, false};
    carve(real, w, m, n, bb + ctx->oversample, nrec_max, true);
  } else {
    RUTV_TRY(prepare(ctx, w, m, n, bb + ctx->oversample, nrec_max, true));
  }
  if (flags & RANDUTV_CHECK_FINITE) RUTV_TRY(check_finite(ctx, L, w, m, n, A, lda));
  RUTV_TRY(start_status(ctx, w));
  RUTV_CUDA(cudaMemcpy2DAsync(w.Twork, m * 8, A, lda * 8, m * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (uv) RUTV_TRY(launch_set_identity(L, n, n, V, ldv));
  Problem P{m, n, bb, q, seed, w.Twork, m, nullptr, m, uv ? V : nullptr, ldv, uv,
            ctx->side_launch(), ctx->eR, ctx->eF, vstream_launch(ctx), ctx->eWv, ctx->eV};
  P.eS = ctx->eS;
  P.eFuv = ctx->eFuv;
  P.reorth = (flags & RANDUTV_REORTH) != 0;
  P.os = ctx->oversample;
  if (!adaptive) {
    RUTV_TRY(run_loop(L, w, P, K, with_final));
  } else {
    double a2 = 0.0;
    RUTV_TRY(launch_sumsq(L, m, n, w.Twork, m, w.red, w.scal));
    RUTV_CUDA(cudaMemcpyAsync(&a2, w.scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
    const double thr2 = tol * tol * a2;
    i64 done = nsamp;
    for (i64 i = 0; i < nsamp; ++i) {
      RUTV_TRY(sampled_step(L, w, P, i));
      // ||T(k':m, k':n)||^2, k' = (i+1) b: disjoint from the side stream's folds
      // of step i (row and column block i)
      const i64 kp = (i + 1) * bb;
      double t2 = 0.0;
      RUTV_TRY(launch_sumsq(L, m - kp, n - kp, w.Twork + kp + kp * m, m, w.red, w.scal));
      RUTV_CUDA(cudaMemcpyAsync(&t2, w.scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
      if (t2 <= thr2) {
        done = i + 1;
        break;
      }
    }
    K = done;
    with_final = done == nsamp;
    if (with_final) RUTV_TRY(final_step(L, w, P, nsamp));
    RUTV_TRY(wait_if(L.stream, P.eF, P.rec_f));
    RUTV_TRY(wait_if(L.stream, P.eFuv, P.rec_fuv));
    if (P.V && P.vl.stream) RUTV_TRY(wait_if(L.stream, P.eV, P.rec_v));
    k = with_final ? n : K * bb;
  }
  const i64 nrec = uv ? K + (with_final ? 1 : 0) : 0;
  // rho = ||T(k:m, k:n)||_F
  RUTV_TRY(launch_sumsq(L, m - k, n - k, w.Twork + k + k * m, m, w.red, w.scal));
  // Tk = T(0:k, :)
  RUTV_CUDA(cudaMemcpy2DAsync(Tk, ldt * 8, w.Twork, m * 8, k * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (uv) RUTV_TRY(backward_uk(L, w, m, n, bb, nrec, with_final, k, Uk, ldu));
  double ss = 0.0;
  RUTV_CUDA(cudaMemcpyAsync(&ss, w.scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  double s2 = 0.0;
  bool squared = false;
  int spec_st = 0x7f7f7f7f;
  if (resid_2 && k < n) {
    Carver rc{(char*)ctx->ws, 0, ctx->ws_bytes, false};
    Work wdummy;
    carve(rc, wdummy, m, n, bb + ctx->oversample, nrec_max, true);
    carve_spec(rc, sw, m - k, n - k);
    RUTV_TRY(spectral_norm(L, sw, m - k, n - k, w.Twork + k + k * m, m, seed, &squared));
    RUTV_CUDA(cudaMemcpyAsync(&s2, sw.d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RUTV_CUDA(cudaMemcpyAsync(&spec_st, sw.status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  }
  const int st = finish(ctx, w);
  *resid_fro = std::sqrt(ss);
  if (resid_2) {
    *resid_2 = k < n ? (squared ? std::sqrt(s2 > 0.0 ? s2 : 0.0) : s2) : 0.0;
    // a non-converged Jacobi SVD of the Rayleigh-Ritz problem: no estimate
    if (spec_st != 0x7f7f7f7f) *resid_2 = -1.0;
  }
  if (k_out) *k_out = k;
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

}  // namespace

extern "C" {

RANDUTV_API int randutv_factor_rank(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, int64_t k,
                                    int64_t b, int q, uint64_t seed, unsigned flags, double* Uk, int64_t ldu,
                                    double* Tk, int64_t ldt, double* V, int64_t ldv, double* resid_fro,
                                    double* resid_2) {
  RUTV_TRY(begin_call(ctx));
  const bool uv = !(flags & RANDUTV_NO_UV);
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A) return -4;
  if (lda < m) return -5;
  if (k < 1 || k > n) return -6;
  if (b < 1) return -7;
  if (q < 0) return -8;
  if (uv && !Uk) return -11;
  if (uv && ldu < m) return -12;
  if (!Tk) return -13;
  if (ldt < k) return -14;
  if (uv && !V) return -15;
  if (uv && ldv < n) return -16;
  if (!resid_fro) return -17;
  return drain_on_error(ctx, truncated_impl(ctx, m, n, A, lda, k, 0.0, b, q, seed, flags, Uk, ldu, Tk, ldt, V, ldv,
                                            resid_fro, nullptr, resid_2));
}

RANDUTV_API int randutv_factor_tol(randutv_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, double tol,
                                   int64_t b, int q, uint64_t seed, unsigned flags, double* Uk, int64_t ldu,
                                   double* Tk, int64_t ldt, double* V, int64_t ldv, int64_t* k_out,
                                   double* resid_fro) {
  RUTV_TRY(begin_call(ctx));
  const bool uv = !(flags & RANDUTV_NO_UV);
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A) return -4;
  if (lda < m) return -5;
  if (!(tol > 0.0)) return -6;
  if (b < 1) return -7;
  if (q < 0) return -8;
  if (uv && !Uk) return -11;
  if (uv && ldu < m) return -12;
  if (!Tk) return -13;
  if (ldt < n) return -14;
  if (uv && !V) return -15;
  if (uv && ldv < n) return -16;
  if (!k_out) return -17;
  if (!resid_fro) return -18;
  return drain_on_error(
      ctx, truncated_impl(ctx, m, n, A, lda, 0, tol, b, q, seed, flags, Uk, ldu, Tk, ldt, V, ldv, resid_fro, k_out));
}

// ----------------------------------------------------------------- literal form

static std::mutex g_lit_mu;
static randutv_ctx* g_lit_ctx[64];
// one literal call per device at a time: the internal ctx's workspace, staging
// buffers and streams are shared by every caller on that device
static std::mutex g_lit_call_mu[64];

static int literal_ctx(randutv_ctx** out) {
  int dev = 0;
  RUTV_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return RANDUTV_ERR_CTX;
  std::lock_guard<std::mutex> lk(g_lit_mu);
  if (!g_lit_ctx[dev]) RUTV_TRY(randutv_create(&g_lit_ctx[dev], dev, nullptr));
  *out = g_lit_ctx[dev];
  return 0;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

RANDUTV_API int randutv_factor(int64_t m, int64_t n, const double* A, int64_t lda, int64_t b, int q, uint64_t seed,
                               double* U, double* T, double* V) {
  if (n < 1) return -2;
  if (m < n) return -1;
  if (!A) return -3;
  if (lda < m) return -4;
  if (b < 1) return -5;
  if (q < 0) return -6;
  if (!U) return -8;
  if (!T) return -9;
  if (!V) return -10;
  randutv_ctx* ctx = nullptr;
  RUTV_TRY(literal_ctx(&ctx));
  std::lock_guard<std::mutex> call_lock(g_lit_call_mu[ctx->device]);
  const bool dev = is_device_ptr(A);
  if (dev != is_device_ptr(T) || dev != is_device_ptr(U) || dev != is_device_ptr(V)) return -9;
  if (dev) return randutv_factor_ex(ctx, m, n, A, lda, b, q, seed, 0u, U, m, T, m, V, n);
  // host pointers: stage through device memory (A -> dT in place, U, V)
  const size_t need = ((size_t)m * n + (size_t)m * m + (size_t)n * n) * sizeof(double);
  if (ctx->stage_bytes < need) {
    if (ctx->stage) cudaFree(ctx->stage);
    ctx->stage = nullptr;
    ctx->stage_bytes = 0;
    cudaError_t e = cudaMalloc(&ctx->stage, need);
    if (e != cudaSuccess) {
      rutv::set_last_error("cudaMalloc(stage)", e);
      cudaGetLastError();
      return RANDUTV_ERR_ALLOC;
    }
    ctx->stage_bytes = need;
  }
  double* dT = ctx->stage;
  double* dU = dT + (size_t)m * n;
  double* dV = dU + (size_t)m * m;
  RUTV_CUDA(cudaMemcpy2DAsync(dT, m * 8, A, lda * 8, m * 8, n, cudaMemcpyHostToDevice, ctx->stream));
  ctx->stats.h2d_bytes += (int64_t)m * n * 8;
  // pinned outputs: column blocks drain to the host during the factorisation
  auto pinned = [](const void* p) {
    cudaPointerAttributes a;
    const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  Drain dr{T, U, V, 0};
  const bool drain = pinned(T) && pinned(U) && pinned(V);
  int st = factor_ex_impl(ctx, m, n, dT, m, b, q, seed, 0u, dU, m, dT, m, dV, n, drain ? &dr : nullptr);
  if (st < 0 || st >= RANDUTV_ERR_BASE) {
    // no drain copy may still be writing the caller's buffers after return
    cudaStreamSynchronize(ctx->stream);
    if (ctx->cps) cudaStreamSynchronize(ctx->cps);
    if (ctx->side) cudaStreamSynchronize(ctx->side);
    if (ctx->vstr) cudaStreamSynchronize(ctx->vstr);
    return st;
  }
  const i64 c0 = drain ? dr.drained : 0;  // columns still on the device
  RUTV_CUDA(cudaMemcpyAsync(T + c0 * m, dT + c0 * m, (size_t)m * (n - c0) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RUTV_CUDA(cudaMemcpyAsync(U + c0 * m, dU + c0 * m, (size_t)m * (m - c0) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RUTV_CUDA(cudaMemcpyAsync(V + c0 * n, dV + c0 * n, (size_t)n * (n - c0) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->stats.d2h_bytes += (int64_t)((size_t)m * n + (size_t)m * m + (size_t)n * n) * 8;
  return st;
}

// --------------------------------------------------------------- step entries

RANDUTV_API int randutv_gaussian(randutv_ctx* ctx, uint64_t seed, int64_t it, int64_t rows, int64_t cols, double* G,
                                 int64_t ldg) {
  RUTV_TRY(begin_call(ctx));
  if (it < 0) return -3;
  if (rows < 0) return -4;
  if (cols < 0) return -5;
  if (!G && rows * cols > 0) return -6;
  if (ldg < rows || ldg < 1) return -7;
  Launch L = ctx->launch();
  RUTV_TRY(launch_gaussian(L, seed, it, rows, cols, G, ldg));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->prof.on) ctx->prof.collect();
  return 0;
}

RANDUTV_API int randutv_dgemm_plan(int64_t M, int64_t N, int64_t K, int64_t ws_elems, int sms, int tail_split,
                                   int64_t* plan) {
  return dgemm_plan(M, N, K, ws_elems, sms, tail_split, plan);
}

RANDUTV_API int randutv_dgemm(randutv_ctx* ctx, int transa, int transb, int64_t M, int64_t N, int64_t K,
                              double alpha, const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                              double* C, int64_t ldc) {
  RUTV_TRY(begin_call(ctx));
  if (transa != 0 && transa != 1) return -2;
  if (transb != 0 && transb != 1) return -3;
  if (M < 0) return -4;
  if (N < 0) return -5;
  if (K < 0) return -6;
  const i64 arows = transa ? K : M, brows = transb ? N : K;
  if (lda < (arows > 1 ? arows : 1)) return -9;
  if (ldb < (brows > 1 ? brows : 1)) return -11;
  if (ldc < (M > 1 ? M : 1)) return -14;
  Launch L = ctx->launch();
  // split-K scratch from the workspace
  const size_t need = (size_t)4 * (size_t)(M > 0 ? M : 1) * (size_t)(N > 0 ? N : 1) * 8 + (1 << 20);
  RUTV_TRY(ensure_ws(ctx, need));
  RUTV_TRY(launch_dgemm(L, transa != 0, transb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                        (double*)ctx->ws, (i64)(ctx->ws_bytes / 8)));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->prof.on) ctx->prof.collect();
  return 0;
}

RANDUTV_API int randutv_panel_qr(randutv_ctx* ctx, int64_t h, int64_t wdt, double* P, int64_t ldp, double* tau,
                                 double* Tf, int64_t ldtf) {
  RUTV_TRY(begin_call(ctx));
  if (wdt < 1) return -3;
  if (h < wdt) return -2;
  if (!P) return -4;
  if (ldp < h) return -5;
  if (!tau) return -6;
  if (!Tf) return -7;
  if (ldtf < wdt) return -8;
  Launch L = ctx->launch();
  Work w;
  RUTV_TRY(prepare(ctx, w, h, wdt, wdt, 0, false));
  RUTV_TRY(panel_qr(L, h, wdt, P, ldp, tau, w.Wu, h, Tf, ldtf, w.qw));
  RUTV_CUDA(cudaStreamSynchronize(ctx->stream));
  RUTV_CUDA(cudaGetLastError());
  if (ctx->prof.on) ctx->prof.collect();
  return 0;
}

RANDUTV_API int randutv_small_svd(randutv_ctx* ctx, int64_t wdt, const double* B, int64_t ldb, double* Us, double* d,
                                  double* Vs) {
  RUTV_TRY(begin_call(ctx));
  if (wdt < 1) return -2;
  if (!B) return -3;
  if (ldb < wdt) return -4;
  if (!Us) return -5;
  if (!d) return -6;
  if (!Vs) return -7;
  Launch L = ctx->launch();
  Work w;
  RUTV_TRY(prepare(ctx, w, wdt, wdt, wdt, 0, false));
  RUTV_TRY(start_status(ctx, w));
  RUTV_TRY(launch_jacobi_svd(L, wdt, B, ldb, Us, d, Vs, w.status, 1, w.jac, w.jac_elems));
  return finish(ctx, w);
}

}  // extern "C"
