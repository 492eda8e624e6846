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
// running argmax; lanes hold rows lane + 32 t of one column at a time.  One
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

RANDUTV_API int randutv_hqrrp(randutv_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, int64_t b,
                              uint64_t seed, unsigned flags, int64_t* jpvt, double* Q, int64_t ldq) {
  RUTV_TRY(begin_call(ctx));
  const bool bq = !(flags & RANDUTV_NO_UV);
  if (n < 1) return -3;
  if (m < n) return -2;
  if (!A) return -4;
  if (lda < m) return -5;
  if (b < 1) return -6;
  if (!jpvt) return -8;
  if (bq && !Q) return -9;
  if (bq && ldq < m) return -10;
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
  for (i64 k = 0; k < n && st == 0; k += bb, ++i) {
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
  st = finish(ctx, w);
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

}  // extern "C"
