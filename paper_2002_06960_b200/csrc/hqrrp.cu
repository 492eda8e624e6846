// HQRRP: blocked randomized column-pivoted Householder QR, A P = Q R
// (Sec. 2 of the paper).  Step i (k = i b,
// r = m - k, s = n - k, w = min(b, s)):
//   H1/H2  Y = G^T R(k:m, k:n)            (b x s; G = randUTV's draw of step i)
//   H3     w steps of Businger-Golub CPQR of Y      -> pivot columns (cpqr_sketch_kernel)
//   H4     the swap-convention permutation of columns k:n of R (all m rows) and
//          of jpvt -- only the <= 2w columns that move are copied
//   H5     unpivoted Householder QR of R(k:m, k:k+w)  (the randUTV panel QR)
//   H6     R(k:m, k+w:n) := Q22^T R(k:m, k+w:n);  Q(:, k:m) := Q(:, k:m) Q22
// H2, H5 and H6 are the DMMA GEMM / panel-QR kernels of the randUTV path; the
// sketch CPQR is the one new kernel.
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>
#include <cooperative_groups.h>

#include "driver.cuh"

namespace cg = cooperative_groups;

namespace rutv {
namespace {

#ifndef RUTV_CP_COLS
#define RUTV_CP_COLS 2
#endif
#ifndef RUTV_CP_NB
#define RUTV_CP_NB 2
#endif
#ifndef RUTV_CP_MINB
#define RUTV_CP_MINB 1
#endif
constexpr int CP_NB = RUTV_CP_NB;
constexpr int CP_THREADS = 256;
constexpr int CP_WARPS = CP_THREADS / 32;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// (a, ca) beats (b, cb): larger squared norm, ties -> lower column (oracle A27)
__device__ __forceinline__ bool beats(double a, int ca, double b, int cb) { return a > b || (a == b && ca < cb); }

__device__ __forceinline__ void warp_argmax(double& v, int& c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oc = __shfl_xor_sync(0xffffffffu, c, o);
    if (beats(ov, oc, v, c)) {
      v = ov;
      c = oc;
    }
  }
}

// H3: `steps` steps of CPQR of Y (rows x s, column-major, ld ldy), rows <= 32 RPL.
// Warp gw owns the columns c with c % NW == gw and keeps no state but its
// running argmax; lanes hold rows lane + 32 t of CP_NB columns at a time.  One
// grid barrier per step: the CTA argmax partials are exchanged through
// part_* (double-buffered by step parity), then every CTA recomputes the
// pivot's reflector (dlarfg, P:337-339 / oracle.hqrrp.cpqr_sketch) from the
// pivot column in global memory and applies it to its own columns, whose
// squared norms of rows j+1: give the next step's candidates.  Columns are
// never moved: piv[j] is the Y column chosen at step j; the swap-convention
// permutation is built afterwards (hq_swap_kernel).
template <int RPL>
__global__ void __launch_bounds__(CP_THREADS, RUTV_CP_MINB) cpqr_sketch_kernel(int rows, int s, int steps, double* __restrict__ Y,
                                                                 i64 ldy, double* part_val, int* part_col,
                                                                 int* __restrict__ piv,
                                                                 unsigned char* __restrict__ done) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int NW = G * CP_WARPS, gw = blockIdx.x * CP_WARPS + warp;
  __shared__ double v[32 * RPL];
  __shared__ double s_tau;
  __shared__ int s_p;
  __shared__ double wv[CP_WARPS];
  __shared__ int wc[CP_WARPS];

  double best = -1.0;
  int bestc = INT_MAX;
  for (int c = gw; c < s; c += NW) {
    const double* y = Y + (i64)c * ldy;
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int r = lane + 32 * t;
      if (r < rows) {
        const double x = y[r];
        acc += x * x;
      }
    }
    acc = warp_sum_d(acc);
    if (beats(acc, c, best, bestc)) {
      best = acc;
      bestc = c;
    }
  }

#ifdef RUTV_CP_PROF
  long long pc[4] = {0, 0, 0, 0}, t0 = clock64(), t1;
#define CP_MARK(i) do { t1 = clock64(); pc[i] += t1 - t0; t0 = t1; } while (0)
#else
#define CP_MARK(i) do { } while (0)
#endif
  for (int j = 0; j < steps; ++j) {
    if (lane == 0) {
      wv[warp] = best;
      wc[warp] = bestc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bv = wv[0];
      int bc = wc[0];
      for (int q = 1; q < CP_WARPS; ++q)
        if (beats(wv[q], wc[q], bv, bc)) {
          bv = wv[q];
          bc = wc[q];
        }
      part_val[(j & 1) * G + blockIdx.x] = bv;
      part_col[(j & 1) * G + blockIdx.x] = bc;
    }
    CP_MARK(0);
    grid.sync();
    CP_MARK(1);
    // global argmax: every thread reads <= ceil(G / CP_THREADS) partials (one
    // L2 round trip), then warp and CTA reductions
    {
      double bv = -1.0;
      int bc = INT_MAX;
#pragma unroll 4
      for (int g = threadIdx.x; g < G; g += CP_THREADS) {
        const double pv = __ldcg(part_val + (j & 1) * G + g);
        const int pc = __ldcg(part_col + (j & 1) * G + g);
        if (beats(pv, pc, bv, bc)) {
          bv = pv;
          bc = pc;
        }
      }
      warp_argmax(bv, bc);
      // (wv / wc of the partial-write phase were consumed before grid.sync)
      if (lane == 0) {
        wv[warp] = bv;
        wc[warp] = bc;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double bv = lane < CP_WARPS ? wv[lane] : -1.0;
      int bc = lane < CP_WARPS ? wc[lane] : INT_MAX;
      warp_argmax(bv, bc);
      const int p = bc;
      // dlarfg of the pivot column's rows j:rows (oracle.householder.dlarfg)
      const double* y = Y + (i64)p * ldy;
      double x[RPL];
      double xn = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int r = lane + 32 * t;
        x[t] = (r > j && r < rows) ? __ldcg(y + r) : 0.0;
        xn += x[t] * x[t];
      }
      xn = warp_sum_d(xn);
      const double alpha = __ldcg(y + j);
      double tau = 0.0, den = 1.0;
      if (xn != 0.0) {
        const double beta = -copysign(hypot(alpha, sqrt(xn)), alpha);
        tau = (beta - alpha) / beta;
        den = alpha - beta;
      }
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int r = lane + 32 * t;
        v[r] = (r == j) ? 1.0 : ((r > j && r < rows) ? x[t] / den : 0.0);
      }
      if (lane == 0) {
        s_tau = tau;
        s_p = p;
        if (blockIdx.x == 0) piv[j] = p;
      }
    }
    __syncthreads();
    CP_MARK(2);
    const int p = s_p;
    const double tau = s_tau;
    if (p % NW == gw && lane == 0) done[p] = 1;
    __syncwarp();
    best = -1.0;
    bestc = INT_MAX;
    if (j + 1 == steps) break;  // the last pivot needs no update
    // CP_NB columns per batch: their done flags and rows are loaded together
    // (done columns are loaded too and then ignored), one L2 round trip per batch
    for (int c0 = gw; c0 < s; c0 += CP_NB * NW) {
      double yr[CP_NB][RPL];
      bool act[CP_NB];
#pragma unroll
      for (int u = 0; u < CP_NB; ++u) {
        const int c = c0 + u * NW;
        const bool in = c < s;
        act[u] = in && c != p && !done[in ? c : 0];
        const double* y = Y + (i64)(in ? c : 0) * ldy;
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int r = lane + 32 * t;
          yr[u][t] = (in && r >= j && r < rows) ? y[r] : 0.0;
        }
      }
      double dot[CP_NB];
#pragma unroll
      for (int u = 0; u < CP_NB; ++u) {
        dot[u] = 0.0;
#pragma unroll
        for (int t = 0; t < RPL; ++t) dot[u] += v[lane + 32 * t] * yr[u][t];
      }
#pragma unroll
      for (int u = 0; u < CP_NB; ++u) dot[u] = warp_sum_d(dot[u]);
      double nn[CP_NB];
#pragma unroll
      for (int u = 0; u < CP_NB; ++u) {
        nn[u] = 0.0;
        const int c = c0 + u * NW;
        double* y = Y + (i64)(c < s ? c : 0) * ldy;
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int r = lane + 32 * t;
          if (act[u] && r >= j && r < rows) {
            if (tau != 0.0) {
              yr[u][t] -= tau * (v[r] * dot[u]);
              y[r] = yr[u][t];
            }
            if (r > j) nn[u] += yr[u][t] * yr[u][t];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < CP_NB; ++u) nn[u] = warp_sum_d(nn[u]);
#pragma unroll
      for (int u = 0; u < CP_NB; ++u) {
        const int c = c0 + u * NW;
        if (act[u] && beats(nn[u], c, best, bestc)) {
          best = nn[u];
          bestc = c;
        }
      }
    }
    CP_MARK(3);
  }
#ifdef RUTV_CP_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("cpqr_prof G=%d s=%d steps=%d reduce %.0f sync %.0f pivot %.0f update %.0f cycles/step\n", G, s, steps,
           (double)pc[0] / steps, (double)pc[1] / steps, (double)pc[2] / steps, (double)pc[3] / steps);
#endif
}

template <int RPL>
int launch_cpqr_t(const Launch& L, int rows, int s, int steps, double* Y, i64 ldy, double* part_val, int* part_col,
                  int* piv, unsigned char* done, int gmax) {
  static int occ = -1;
  if (occ < 0) {
    RUTV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cpqr_sketch_kernel<RPL>, CP_THREADS, 0));
    if (occ < 1) occ = 1;
  }
  int G = (s + CP_WARPS * RUTV_CP_COLS - 1) / (CP_WARPS * RUTV_CP_COLS);  // >= RUTV_CP_COLS columns per warp
  G = G < 1 ? 1 : G;
  static int occ_cap = -1;
  if (occ_cap < 0) {
    const char* e = getenv("RUTV_HQ_CPQR_OCC");
    occ_cap = e ? atoi(e) : 0;
  }
  const int oc = (occ_cap > 0 && occ_cap < occ) ? occ_cap : occ;
  G = G > oc * L.device_sms ? oc * L.device_sms : G;
  G = G > gmax ? gmax : G;
  void* args[] = {&rows, &s, &steps, &Y, &ldy, &part_val, &part_col, &piv, &done};
  const size_t pe = L.pbegin();
  RUTV_CUDA(cudaLaunchCooperativeKernel((void*)cpqr_sketch_kernel<RPL>, dim3(G), dim3(CP_THREADS), args, 0,
                                        L.stream));
  L.count();
  // algorithmic: the b x s sketch read + written once per step (rows j:b)
  L.pend(PK_OTHER, 4.0 * rows * (double)s * steps, 8.0 * 2.0 * rows * (double)s * steps / 2.0, pe);
  return 0;
}

// H4 helpers: perm (position -> Y column) and inv start as the identity; the
// w recorded pivots are replayed as swaps (LAPACK dgeqp3's convention).
__global__ void hq_iota_kernel(int s, int* perm, int* inv, int* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s; i += gridDim.x * blockDim.x) {
    perm[i] = i;
    inv[i] = i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = 0;
}

__global__ void hq_swap_kernel(int steps, const int* __restrict__ piv, int* perm, int* inv) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int j = 0; j < steps; ++j) {
    const int p = piv[j];
    const int pp = inv[p];
    if (pp != j) {
      const int cj = perm[j];
      perm[j] = p;
      perm[pp] = cj;
      inv[p] = j;
      inv[cj] = pp;
    }
  }
}

__global__ void hq_collect_kernel(int s, const int* __restrict__ perm, int* cnt, int* moved) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s; i += gridDim.x * blockDim.x)
    if (perm[i] != i) moved[atomicAdd(cnt, 1)] = i;
}

// tmp(:, t) := X(:, perm[moved[t]]) for t < *cnt (and the jpvt entries)
__global__ void hq_gather_kernel(i64 m, const double* __restrict__ X, i64 ldx, const int* __restrict__ perm,
                                 const int* __restrict__ cnt, const int* __restrict__ moved, double* __restrict__ tmp,
                                 const int64_t* __restrict__ jp, int64_t* __restrict__ jtmp) {
  const int t = blockIdx.y;
  if (t >= *cnt) return;
  const int src = perm[moved[t]];
  const double* x = X + (i64)src * ldx;
  double* d = tmp + (i64)t * m;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (i64)gridDim.x * blockDim.x) d[r] = x[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) jtmp[t] = jp[src];
}

__global__ void hq_scatter_kernel(i64 m, double* __restrict__ X, i64 ldx, const int* __restrict__ cnt,
                                  const int* __restrict__ moved, const double* __restrict__ tmp,
                                  int64_t* __restrict__ jp, const int64_t* __restrict__ jtmp) {
  const int t = blockIdx.y;
  if (t >= *cnt) return;
  const int dst = moved[t];
  double* x = X + (i64)dst * ldx;
  const double* sp = tmp + (i64)t * m;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (i64)gridDim.x * blockDim.x) x[r] = sp[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) jp[dst] = jtmp[t];
}

__global__ void hq_jpvt_init_kernel(i64 n, int64_t* jp) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) jp[i] = i;
}

struct HqWork {
  double* part_val;
  int* part_col;
  int* piv;
  int* perm;
  int* inv;
  int* cnt;
  int* moved;
  unsigned char* done;
  int64_t* jtmp;
  int gmax;
  // Q stream (the Q update of step i overlaps step i+1): second (W, T) buffer
  // and the stream's own GEMM temporaries
  double *Wu2, *TU2, *Zq, *Zq2, *gq;
};

void carve_hq(Carver& c, HqWork& h, i64 n, i64 b) {
  h.gmax = 8 * 148;
  h.part_val = c.take<double>(2 * h.gmax);
  h.part_col = c.take<int>(2 * h.gmax);
  h.piv = c.take<int>(b);
  h.perm = c.take<int>(n);
  h.inv = c.take<int>(n);
  h.cnt = c.take<int>(4);
  h.moved = c.take<int>(2 * b);
  h.done = c.take<unsigned char>(n);
  h.jtmp = c.take<int64_t>(2 * b);
}

void carve_hq_q(Carver& c, HqWork& h, i64 m, i64 b) {
  h.Wu2 = c.take<double>(m * b);
  h.TU2 = c.take<double>(b * b);
  h.Zq = c.take<double>(m * b);
  h.Zq2 = c.take<double>(m * b);
  h.gq = c.take<double>(4 * m * b);
}

bool hq_qstream_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_HQ_QSTREAM");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

int launch_cpqr(const Launch& L, int rows, int s, int steps, double* Y, i64 ldy, const HqWork& h) {
  const int rpl = (rows + 31) / 32;
  if (rpl <= 1) return launch_cpqr_t<1>(L, rows, s, steps, Y, ldy, h.part_val, h.part_col, h.piv, h.done, h.gmax);
  if (rpl <= 2) return launch_cpqr_t<2>(L, rows, s, steps, Y, ldy, h.part_val, h.part_col, h.piv, h.done, h.gmax);
  if (rpl <= 4) return launch_cpqr_t<4>(L, rows, s, steps, Y, ldy, h.part_val, h.part_col, h.piv, h.done, h.gmax);
  if (rpl <= 8) return launch_cpqr_t<8>(L, rows, s, steps, Y, ldy, h.part_val, h.part_col, h.piv, h.done, h.gmax);
  return launch_cpqr_t<16>(L, rows, s, steps, Y, ldy, h.part_val, h.part_col, h.piv, h.done, h.gmax);
}

// H4: permute the columns k:n of R (m rows) and jpvt(k:n) by the CPQR pivots
int permute_columns(const Launch& L, i64 m, i64 s, int steps, double* Rk, i64 ldr, int64_t* jpk, double* tmp,
                    const HqWork& h) {
  const unsigned gb = (unsigned)std::min<i64>((s + 255) / 256, 4 * 148);
  hq_iota_kernel<<<gb, 256, 0, L.stream>>>((int)s, h.perm, h.inv, h.cnt);
  hq_swap_kernel<<<1, 32, 0, L.stream>>>(steps, h.piv, h.perm, h.inv);
  hq_collect_kernel<<<gb, 256, 0, L.stream>>>((int)s, h.perm, h.cnt, h.moved);
  const dim3 grid((unsigned)std::min<i64>((m + 255) / 256, 64), (unsigned)(2 * steps));
  hq_gather_kernel<<<grid, 256, 0, L.stream>>>(m, Rk, ldr, h.perm, h.cnt, h.moved, tmp, jpk, h.jtmp);
  hq_scatter_kernel<<<grid, 256, 0, L.stream>>>(m, Rk, ldr, h.cnt, h.moved, tmp, jpk, h.jtmp);
  L.count(5);
  RUTV_CHECK_LAUNCH("hqrrp permute");
  return 0;
}

}  // namespace
}  // namespace rutv

using namespace rutv;

extern "C" {

static int hqrrp_impl(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t ktr, int64_t b,
                      uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq, double* resid_fro);

RANDUTV_API int randutv_hqrrp(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t b,
                              uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq) {
  return hqrrp_impl(ctx, m, n, A, lda, -1, b, seed, flags, jpvt, Q, ldq, nullptr);
}

RANDUTV_API int randutv_hqrrp_rank(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t k,
                                   int64_t b, uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq,
                                   double* resid_fro) {
  RUTV_TRY(begin_call(ctx));
  const bool bq = !(flags & RANDUTV_NO_UV);
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A) return -4;
  if (lda < m) return -5;
  if (k < 1 || k > n) return -6;
  if (b < 1 || (b < n ? b : n) > 512) return -7;
  if (!jpvt) return -10;
  if (bq && !Q) return -11;
  if (bq && ldq < m) return -12;
  return hqrrp_impl(ctx, m, n, A, lda, k, b, seed, flags, jpvt, Q, ldq, resid_fro);
}

static int hqrrp_impl(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t ktr, int64_t b,
                      uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq, double* resid_fro) {
  RUTV_TRY(begin_call(ctx));
  const bool bq = !(flags & RANDUTV_NO_UV);
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A) return -4;
  if (lda < m) return -5;
  if (b < 1) return -6;
  if (!jpvt) return -9;
  if (bq && !Q) return -10;
  if (bq && ldq < m) return -11;
  const i64 bb = b < n ? b : n;
  if (bb > 512) return -6;  // the sketch CPQR keeps <= 512 rows per column in registers
  Launch L = ctx->launch();
  Work w;
  HqWork h;
  const bool qs = bq && hq_qstream_on();
  Carver dry{nullptr, 0, 0, true};
  carve(dry, w, m, n, bb, 0, false);
  carve_hq(dry, h, n, bb);
  if (qs) carve_hq_q(dry, h, m, bb);
  RUTV_TRY(ensure_ws(ctx, dry.off));
  Carver real{(char*)ctx->ws, 0, ctx->ws_bytes, false};
  carve(real, w, m, n, bb, 0, false);
  carve_hq(real, h, n, bb);
  if (qs) carve_hq_q(real, h, m, bb);
  if (flags & RANDUTV_CHECK_FINITE) RUTV_TRY(check_finite(ctx, L, w, m, n, A, lda));
  RUTV_TRY(start_status(ctx, w));
  hq_jpvt_init_kernel<<<(unsigned)std::min<i64>((n + 255) / 256, 1024), 256, 0, L.stream>>>(n, jpvt);
  L.count();
  if (bq) RUTV_TRY(launch_set_identity(L, m, m, Q, ldq));
  // Q stream: H6's Q update of step i runs on ctx->vstr (one-shot GEMM tiles)
  // behind step i+1's sketch, CPQR and permutation; (W, T) alternate between
  // two buffers, and step i+2's panel QR waits for the Q update of step i.
  Launch LQ = ctx->v_launch();
  Work wq = w;
  cudaEvent_t eQ[2] = {nullptr, nullptr};
  if (qs) {
    wq.Z = h.Zq;
    wq.Z2 = h.Zq2;
    wq.gemm_ws = h.gq;
    wq.gemm_ws_elems = 4 * m * bb;
    for (auto& e : eQ) RUTV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  int st = 0;
  i64 i = 0;
  const i64 kstop = ktr < 0 ? n : std::min<i64>(n, (ktr + bb - 1) / bb * bb);
  for (i64 k = 0; k < kstop && st == 0; k += bb, ++i) {
    const i64 r = m - k, s = n - k, wd = bb < s ? bb : s;
    const int sel = (int)(i & 1);
    double* Wu = (qs && sel) ? h.Wu2 : w.Wu;
    double* TU = (qs && sel) ? h.TU2 : w.TU;
    double* Rk = A + k * lda;  // columns k:n, all rows
    auto step = [&]() -> int {
      // H1, H2: Y (bb x s, ld bb) = G^T R(k:m, k:n)
      RUTV_TRY(launch_gaussian(L, seed, i, r, bb, w.G, r));
      RUTV_TRY(launch_dgemm(L, true, false, bb, s, r, 1.0, w.G, r, Rk + k, lda, 0.0, w.Y, bb, w.gemm_ws,
                            w.gemm_ws_elems));
      // H3
      RUTV_CUDA(cudaMemsetAsync(h.done, 0, (size_t)s, L.stream));
      RUTV_TRY(launch_cpqr(L, (int)bb, (int)s, (int)wd, w.Y, bb, h));
      // H4
      RUTV_TRY(permute_columns(L, m, s, (int)wd, Rk, lda, jpvt + k, w.Acat, h));
      // H5 (the (W, T) buffer is free once the Q update of step i-2 is done)
      if (qs && i >= 2) RUTV_CUDA(cudaStreamWaitEvent(L.stream, eQ[sel], 0));
      RUTV_TRY(panel_qr(L, r, wd, Rk + k, lda, w.tauU, Wu, r, TU, bb, w.qw));
      RUTV_TRY(launch_triu(L, wd, wd, Rk + k, lda));
      RUTV_TRY(launch_fill(L, r - wd, wd, 0.0, Rk + k + wd, lda));
      // H6
      if (qs) {
        RUTV_CUDA(cudaEventRecord(ctx->eWv, L.stream));
        RUTV_CUDA(cudaStreamWaitEvent(LQ.stream, ctx->eWv, 0));
        RUTV_TRY(apply_right(LQ, wq, m, r, wd, Q + k * ldq, ldq, Wu, r, TU, bb));
        RUTV_CUDA(cudaEventRecord(eQ[sel], LQ.stream));
      }
      if (s > wd) RUTV_TRY(apply_left_t(L, w, r, s - wd, wd, Rk + k + wd * lda, lda, Wu, r, TU, bb));
      if (bq && !qs) RUTV_TRY(apply_right(L, w, m, r, wd, Q + k * ldq, ldq, Wu, r, TU, bb));
      return 0;
    };
    st = step();
  }
  if (qs) {
    // the main stream (and so the caller) must not run ahead of the Q stream
    if (cudaEventRecord(ctx->eV, LQ.stream) != cudaSuccess || cudaStreamWaitEvent(L.stream, ctx->eV, 0) != cudaSuccess)
      st = st ? st : RANDUTV_ERR_CUDA;
    for (auto& e : eQ)
      if (e) cudaEventDestroy(e);
  }
  if (st != 0) {
    cudaStreamSynchronize(L.stream);
    return st;
  }
  if (ktr > 0 && resid_fro) {
    // rho = ||R(k:m, k:n)||_F: the error of the rank-k truncation
    RUTV_TRY(launch_sumsq(L, m - ktr, n - ktr, A + ktr + ktr * lda, lda, w.red, w.scal));
    double ss = 0.0;
    RUTV_CUDA(cudaMemcpyAsync(&ss, w.scal, sizeof(double), cudaMemcpyDeviceToHost, L.stream));
    st = finish(ctx, w);
    *resid_fro = sqrt(ss);
  } else {
    st = finish(ctx, w);
  }
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// HQRRP_left, host-streamed (Sec. 2.3 of the paper): A stays in
// (pinned) host memory and is overwritten by R with the Householder tails
// below the diagonal (LAPACK dgeqp3 layout); only the current
// column block is ever written back.  Iteration i (k = i b, w = min(b, n-k)):
//   L1  Gt = [0; G^(i)] (m x b);  Gt := Q Gt = H_0 (... (H_{i-1} Gt))
//       -- a pass over the stored reflector blocks i-1 .. 0 (rows k_j:m)
//   L2  Y = Gt^T A(:, k:n)  (b x s) -- a pass over the UNMODIFIED remaining
//       columns: Y = G (Q^* A P)(k:m, k:n) = G R22 of the right-looking
//       algorithm ("repeat some of the arithmetic")
//   L3  CPQR of Y (cpqr_sketch_kernel) -> pivots; the <= 2w host columns the
//       swap-convention permutation moves are copied through the device
//   L4  X = A(:, k:k+w);  X := Q^* X  -- a pass over reflector blocks 0 .. i-1
//   L5  Householder QR of X(k:m) (tau, T_i kept on the device); X -> host.
// Panels stream H2D through a two-slot ring (one-panel prefetch on a copy
// stream); the T factors of all blocks stay in HBM (n b doubles).
namespace rutv {
namespace {

__global__ void unit_lower_kernel(i64 rows, i64 cols, const double* __restrict__ P, i64 ldp, double* __restrict__ W,
                                  i64 ldw) {
  const i64 total = rows * cols;
  for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e % rows, c = e / rows;
    W[r + c * ldw] = r > c ? P[r + c * ldp] : (r == c ? 1.0 : 0.0);
  }
}

int launch_unit_lower(const Launch& L, i64 rows, i64 cols, const double* P, i64 ldp, double* W, i64 ldw) {
  if (rows <= 0 || cols <= 0) return 0;
  const unsigned g = (unsigned)std::min<i64>((rows * cols + 255) / 256, 4 * 148);
  unit_lower_kernel<<<g, 256, 0, L.stream>>>(rows, cols, P, ldp, W, ldw);
  L.count();
  RUTV_CHECK_LAUNCH("unit_lower_kernel");
  return 0;
}

struct HostLeft {
  Launch L;
  cudaStream_t h2d = nullptr;
  double* A = nullptr;
  i64 m = 0, n = 0, lda = 0, b = 0;
  double* slot[2] = {nullptr, nullptr};
  cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr}, compdone = nullptr;
  randutv_host_report* rep = nullptr;
  std::vector<cudaEvent_t> pool;  // H2D copy timing (start, end) pairs
  size_t used = 0;
  std::vector<std::pair<size_t, size_t>> spans;
  int mark(cudaStream_t s, size_t* idx) {
    if (used == pool.size()) {
      cudaEvent_t e;
      RUTV_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    RUTV_CUDA(cudaEventRecord(pool[used], s));
    *idx = used++;
    return 0;
  }
  ~HostLeft() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    for (int s = 0; s < 2; ++s) {
      if (ready[s]) cudaEventDestroy(ready[s]);
      if (freed[s]) cudaEventDestroy(freed[s]);
    }
    if (compdone) cudaEventDestroy(compdone);
    if (h2d) cudaStreamDestroy(h2d);
  }
};

struct PanelItem {
  i64 col0, r0, w;  // columns col0 .. col0+w, rows r0 .. m
};

// stream the items H2D through the two slots; f(t, device ptr (ld = m - r0))
template <class F>
int left_pass(HostLeft& H, const std::vector<PanelItem>& items, F&& f) {
  const int N = (int)items.size();
  if (N == 0) return 0;
  // everything the compute stream wrote to host so far lands before the pass reads
  RUTV_CUDA(cudaEventRecord(H.compdone, H.L.stream));
  RUTV_CUDA(cudaStreamWaitEvent(H.h2d, H.compdone, 0));
  auto issue = [&](int t) -> int {
    const int s = t & 1;
    const PanelItem& it = items[t];
    const i64 rows = H.m - it.r0;
    RUTV_CUDA(cudaStreamWaitEvent(H.h2d, H.freed[s], 0));
    size_t e0 = 0, e1 = 0;
    RUTV_TRY(H.mark(H.h2d, &e0));
    RUTV_CUDA(cudaMemcpy2DAsync(H.slot[s], rows * 8, H.A + it.col0 * H.lda + it.r0, H.lda * 8, rows * 8, it.w,
                                cudaMemcpyHostToDevice, H.h2d));
    RUTV_TRY(H.mark(H.h2d, &e1));
    H.spans.push_back({e0, e1});
    RUTV_CUDA(cudaEventRecord(H.ready[s], H.h2d));
    H.rep->h2d_bytes += rows * it.w * 8;
    return 0;
  };
  RUTV_TRY(issue(0));
  for (int t = 0; t < N; ++t) {
    if (t + 1 < N) RUTV_TRY(issue(t + 1));
    const int s = t & 1;
    RUTV_CUDA(cudaStreamWaitEvent(H.L.stream, H.ready[s], 0));
    RUTV_TRY(f(t, H.slot[s]));
    RUTV_CUDA(cudaEventRecord(H.freed[s], H.L.stream));
  }
  return 0;
}

}  // namespace
}  // namespace rutv

extern "C" {

RANDUTV_API int randutv_hqrrp_host(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b,
                                   uint64_t seed, unsigned flags, int64_t* jpvt_host, double* tau_host,
                                   randutv_host_report* report) {
  RUTV_TRY(begin_call(ctx));
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A_host) return -4;
  if (lda < m) return -5;
  if (b < 1) return -6;
  if (flags != 0) return -8;
  if (!jpvt_host) return -9;
  if (!tau_host) return -10;
  const i64 bb = b < n ? b : n;
  if (bb > 512) return -6;
  const i64 nblk = (n + bb - 1) / bb;
  randutv_host_report rep;
  memset(&rep, 0, sizeof(rep));
  Launch L = ctx->launch();
  Work w;
  HqWork h;
  double *slots = nullptr, *Tall = nullptr, *tauall = nullptr, *gath = nullptr;
  auto carve_all = [&](Carver& c) {
    carve(c, w, m, n, bb, 0, false);
    carve_hq(c, h, n, bb);
    slots = c.take<double>(2 * m * bb);
    Tall = c.take<double>(nblk * bb * bb);
    tauall = c.take<double>(n);
    gath = c.take<double>(2 * bb * m);
  };
  Carver dry{nullptr, 0, 0, true};
  carve_all(dry);
  RUTV_TRY(ensure_ws(ctx, dry.off));
  Carver real{(char*)ctx->ws, 0, ctx->ws_bytes, false};
  carve_all(real);
  double* Gt = w.G;   // m x b
  double* Y = w.Y;    // b x s, ld b
  double* X = w.Zf;   // m x b: the current block
  double* Wb = w.Wu;  // explicit unit-lower W of a streamed reflector block
  double* Wx = w.Acat;  // panel_qr's explicit W (unused here)

  bool registered = false;
  {
    cudaPointerAttributes a;
    if (!(cudaPointerGetAttributes(&a, A_host) == cudaSuccess && a.type == cudaMemoryTypeHost)) {
      cudaGetLastError();
      RUTV_CUDA(cudaHostRegister(A_host, (size_t)lda * n * 8, cudaHostRegisterDefault));
      registered = true;
    }
  }
  int st = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  {
    HostLeft H;
    H.L = L;
    H.A = A_host;
    H.m = m;
    H.n = n;
    H.lda = lda;
    H.b = bb;
    H.rep = &rep;
    H.slot[0] = slots;
    H.slot[1] = slots + m * bb;
    auto init = [&]() -> int {
      RUTV_CUDA(cudaStreamCreateWithFlags(&H.h2d, cudaStreamNonBlocking));
      for (int s = 0; s < 2; ++s) {
        RUTV_CUDA(cudaEventCreateWithFlags(&H.ready[s], cudaEventDisableTiming));
        RUTV_CUDA(cudaEventCreateWithFlags(&H.freed[s], cudaEventDisableTiming));
        RUTV_CUDA(cudaEventRecord(H.freed[s], L.stream));
      }
      RUTV_CUDA(cudaEventCreateWithFlags(&H.compdone, cudaEventDisableTiming));
      RUTV_CUDA(cudaEventCreate(&t0));
      RUTV_CUDA(cudaEventCreate(&t1));
      RUTV_CUDA(cudaEventRecord(t0, L.stream));
      return start_status(ctx, w);
    };
    st = init();
    std::vector<int> piv((size_t)bb), perm, inv;
    std::vector<int64_t> jp((size_t)n);
    for (i64 c = 0; c < n; ++c) jp[c] = c;
    i64 i = 0;
    for (i64 k = 0; k < n && st == 0; k += bb, ++i) {
      const i64 r = m - k, s = n - k, wd = bb < s ? bb : s;
      auto iteration = [&]() -> int {
        // L1: Gt = Q [0; G]
        RUTV_TRY(launch_fill(L, k, bb, 0.0, Gt, m));
        RUTV_TRY(launch_gaussian(L, seed, i, r, bb, Gt + k, m));
        std::vector<PanelItem> back, fwd, rest;
        for (i64 j = i - 1; j >= 0; --j) back.push_back({j * bb, j * bb, std::min(bb, n - j * bb)});
        for (i64 j = 0; j < i; ++j) fwd.push_back({j * bb, j * bb, std::min(bb, n - j * bb)});
        for (i64 p = i; p < nblk; ++p) rest.push_back({p * bb, 0, std::min(bb, n - p * bb)});
        RUTV_TRY(left_pass(H, back, [&](int t, double* P) -> int {
          const PanelItem& it = back[t];
          const i64 rj = m - it.r0;
          RUTV_TRY(launch_unit_lower(L, rj, it.w, P, rj, Wb, rj));
          const double* Tj = Tall + (it.col0 / bb) * bb * bb;
          RUTV_TRY(launch_dgemm(L, true, false, it.w, bb, rj, 1.0, Wb, rj, Gt + it.r0, m, 0.0, w.Z, it.w, w.gemm_ws,
                                w.gemm_ws_elems));
          RUTV_TRY(launch_dgemm(L, false, false, it.w, bb, it.w, 1.0, Tj, bb, w.Z, it.w, 0.0, w.Z2, it.w, nullptr, 0));
          return launch_dgemm(L, false, false, rj, bb, it.w, -1.0, Wb, rj, w.Z2, it.w, 1.0, Gt + it.r0, m, nullptr, 0);
        }));
        // L2: Y = Gt^T A(:, k:n)
        RUTV_TRY(left_pass(H, rest, [&](int t, double* P) -> int {
          const PanelItem& it = rest[t];
          return launch_dgemm(L, true, false, bb, it.w, m, 1.0, Gt, m, P, m, 0.0, Y + (it.col0 - k) * bb, bb,
                              w.gemm_ws, w.gemm_ws_elems);
        }));
        // L3: pivots, then the swap-convention permutation of the host columns k:n
        RUTV_CUDA(cudaMemsetAsync(h.done, 0, (size_t)s, L.stream));
        RUTV_TRY(launch_cpqr(L, (int)bb, (int)s, (int)wd, Y, bb, h));
        RUTV_CUDA(cudaMemcpyAsync(piv.data(), h.piv, wd * sizeof(int), cudaMemcpyDeviceToHost, L.stream));
        RUTV_CUDA(cudaStreamSynchronize(L.stream));
        perm.resize((size_t)s);
        inv.resize((size_t)s);
        for (i64 c = 0; c < s; ++c) perm[c] = inv[c] = (int)c;
        for (i64 j = 0; j < wd; ++j) {
          const int p = piv[j], pp = inv[p];
          if (pp != j) {
            const int cj = perm[j];
            perm[j] = p;
            perm[pp] = cj;
            inv[p] = (int)j;
            inv[cj] = pp;
          }
        }
        std::vector<i64> moved;
        for (i64 c = 0; c < s; ++c)
          if (perm[c] != c) moved.push_back(c);
        for (size_t t = 0; t < moved.size(); ++t) {
          RUTV_CUDA(cudaMemcpyAsync(gath + t * m, A_host + (k + perm[moved[t]]) * lda, m * 8, cudaMemcpyHostToDevice,
                                    L.stream));
          rep.h2d_bytes += m * 8;
        }
        for (size_t t = 0; t < moved.size(); ++t) {
          RUTV_CUDA(cudaMemcpyAsync(A_host + (k + moved[t]) * lda, gath + t * m, m * 8, cudaMemcpyDeviceToHost,
                                    L.stream));
          rep.d2h_bytes += m * 8;
        }
        {
          std::vector<int64_t> old(jp.begin() + k, jp.end());
          for (i64 c : moved) jp[k + c] = old[perm[c]];
        }
        // L4: X = Q^* A(:, k:k+w)
        RUTV_CUDA(cudaMemcpy2DAsync(X, m * 8, A_host + k * lda, lda * 8, m * 8, wd, cudaMemcpyHostToDevice, L.stream));
        rep.h2d_bytes += m * wd * 8;
        RUTV_TRY(left_pass(H, fwd, [&](int t, double* P) -> int {
          const PanelItem& it = fwd[t];
          const i64 rj = m - it.r0;
          RUTV_TRY(launch_unit_lower(L, rj, it.w, P, rj, Wb, rj));
          const double* Tj = Tall + (it.col0 / bb) * bb * bb;
          return apply_left_t(L, w, rj, wd, it.w, X + it.r0, m, Wb, rj, Tj, bb);
        }));
        // L5: QR of the block, write back
        RUTV_TRY(panel_qr(L, r, wd, X + k, m, tauall + k, Wx, r, Tall + i * bb * bb, bb, w.qw));
        RUTV_CUDA(cudaMemcpy2DAsync(A_host + k * lda, lda * 8, X, m * 8, m * 8, wd, cudaMemcpyDeviceToHost, L.stream));
        rep.d2h_bytes += m * wd * 8;
        return 0;
      };
      st = iteration();
    }
    if (st == 0) {
      cudaEventRecord(t1, L.stream);
      if (cudaMemcpyAsync(tau_host, tauall, n * 8, cudaMemcpyDeviceToHost, L.stream) != cudaSuccess) st = RANDUTV_ERR_CUDA;
      rep.d2h_bytes += n * 8;
    }
    if (st == 0) st = finish(ctx, w);
    if (st == 0) {
      memcpy(jpvt_host, jp.data(), n * sizeof(int64_t));
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, t0, t1) == cudaSuccess) rep.wall_ms = ms;
      double tot = 0.0;
      for (auto& pr : H.spans) {
        float x = 0.f;
        if (cudaEventElapsedTime(&x, H.pool[pr.first], H.pool[pr.second]) == cudaSuccess) tot += x;
      }
      rep.h2d_ms = tot;
      rep.cache_slots = 2;
      rep.slot_bytes = (int64_t)(m * bb * 8);
    }
    cudaStreamSynchronize(L.stream);
    if (H.h2d) cudaStreamSynchronize(H.h2d);
  }
  if (t0) cudaEventDestroy(t0);
  if (t1) cudaEventDestroy(t1);
  if (registered) cudaHostUnregister(A_host);
  cudaGetLastError();
  ctx->stats.h2d_bytes += rep.h2d_bytes;
  ctx->stats.d2h_bytes += rep.d2h_bytes;
  if (report) *report = rep;
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

}  // extern "C"
