// K3/K4 -- S4 and S6 of SURVEY.md §8(a): unpivoted Householder QR of a tall
// panel and its compact-WY factor.
//
// Paper: "[Y, T_V] := unpivoted_QR(Y)" and "[[A11; A21], T_U] := unpivoted_QR(...)"
// (Fig. fig:FLArandutv), with W_V / W_U "the unit
// lower trapezoidal matrices stored below the diagonal" and the
// transforms applied as X - X W T W^T.  Sec. 3.1 steps 1-2
// (P:570-582).  Conventions (reading A9): LAPACK dlarfg
// reflectors -- xi = ||x'||; xi == 0 -> tau = 0; else beta = -sign(alpha)
// hypot(alpha, xi), tau = (beta - alpha)/beta, v = (1, x'/(alpha - beta)) -- and
// the dlarft forward/columnwise factor, Q = H_1...H_w = I - W T W^T.
//
// Structure (right-looking blocked QR with leaf width NB = 32):
//   for each leaf L of NB columns:
//     qr_leaf_kernel   cooperative grid over the panel rows.  Per column: ONE
//                      grid-wide barrier.  Each CTA forms, over its rows, the
//                      partial ||x'||^2 and the partial dots x'.P(:,l) of the
//                      *unscaled* column with the later leaf columns; after the
//                      barrier every CTA reduces the partials in the same fixed
//                      order (bitwise identical beta, tau, w in every CTA) and
//                      updates its own rows, so no second barrier is needed.
//                      The NB x NB top block is replicated in every CTA's
//                      shared memory and updated identically by all of them.
//                      It also writes the leaf's explicit W columns (unit
//                      diagonal, zeros above) -- no separate extraction pass.
//     S = W^T W_L      DMMA GEMM (K = h - c0, split-K)
//     t_block          T_L from S_LL and tau (dlarft recurrence, one warp) and
//                      T(0:c0, L) = -T(0:c0,0:c0) S(0:c0, L) T_L, one CTA
//     trailing update  P(c0:h, L+:) -= W_L T_L^T (W_L^T P(c0:h, L+:))  (3 GEMMs)
// The leaf kernel is bound by L2 latency and the per-column barrier; the
// GEMMs carry the O(h w^2) flops.  All reductions are fixed-order, so the
// factorisation is bitwise deterministic (required for the redundant QR(Y) on
// every rank of the multi-GPU layout).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int NB = 32;
constexpr int LEAF_THREADS = 256;
constexpr int LEAF_MAX_CTAS = 128;
constexpr int PSTRIDE = NB + 1;  // partial record: [0] = ||x'||^2, [1+l] = x'.P(:,l)
constexpr int PREC = PSTRIDE + 1;  // its stride in global memory (even: 16-byte copies)
// leaf record area: 2 parities x 128 CTAs x PREC (grid leaf)
constexpr long long LEAF_REC_ELEMS = 2LL * LEAF_MAX_CTAS * PREC;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// DSMEM push exchange (cluster leaf, PUSH): each CTA stores its partial
// record straight into every CTA's inbox with st.async, which completes bytes
// on the receiver's mbarrier; the receiver waits on its own barrier -- one
// remote-store latency per column instead of a cluster barrier + DSMEM loads.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Per-column register work of the leaf with the column index J a template
// argument (v[k][J] must be a compile-time register index).  Dispatched by a
// switch -- an indexed branch -- instead of an unrolled scan comparing jj with
// all 32 indices (the compare chain carried ~10 % of the leaf's stall samples).
template <int J, int R>
__device__ __forceinline__ void leaf_partials(const double (&v)[R > 0 ? R : 1][NB], double (&acc)[PSTRIDE]) {
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double x = v[k][J];
    acc[0] = fma(x, x, acc[0]);
#pragma unroll
    for (int l = J + 1; l < NB; ++l) acc[1 + l] = fma(x, v[k][l], acc[1 + l]);
  }
}
template <int J, int R>
__device__ __forceinline__ void leaf_update(double (&v)[R > 0 ? R : 1][NB], double scal, double t,
                                            const double* __restrict__ wv) {
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double vv = v[k][J] * scal;
    v[k][J] = vv;
    const double tv = t * vv;
#pragma unroll
    for (int l = J + 1; l < NB; ++l) v[k][l] = fma(-tv, wv[l], v[k][l]);
  }
}
#define RUTV_CASES32(F) \
  F(0) F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) F(12) F(13) F(14) F(15) F(16) F(17) F(18) F(19) \
  F(20) F(21) F(22) F(23) F(24) F(25) F(26) F(27) F(28) F(29) F(30) F(31)

// P points at the panel's top-left element (row 0, col 0); the leaf is columns
// [c0, c0+nb), rows [c0, h).  Rows [c0, c0+nb) form the replicated top block;
// rows [c0+nb, h) are split into contiguous slabs, one per CTA.  R > 0: each
// thread keeps its R slab rows of the 32 leaf columns in registers for the whole
// leaf (one read and one write of the slab); R == 0: rows stay in global memory
// (L2) -- for panels taller than 128 x 256 x 2 rows.
// CLUSTER: the G (<= 16) CTAs form one thread-block cluster; the per-column
// exchange is a cluster barrier + DSMEM reads of the other CTAs' records
// (tools/sync_micro.cu: ~1.0 us for 16 CTAs) instead of a grid barrier + an L2
// round trip through `partials` (~3.6 us for 64 CTAs).
// S > 0 (cluster leaves only): each thread also keeps S more rows of the slab
// in shared memory (dynamic, column-major with ld S*256 so a warp's row
// accesses are consecutive), so one 16-CTA cluster holds panels of up to
// 16 * 256 * (R + S) rows and the per-column exchange stays a cluster barrier
// + DSMEM instead of a grid barrier + L2 round trips (c3's 16384-row panels:
// R = 2, S = 2).
template <int R, bool CLUSTER, int S = 0, bool PUSH = false>
__global__ void __launch_bounds__(LEAF_THREADS, 1)
    qr_leaf_kernel(double* __restrict__ P, i64 h, i64 ldp, i64 c0, int nb, double* __restrict__ tau,
                   double* __restrict__ partials, double* __restrict__ Wx, i64 ldw) {
  __shared__ double mine[2][PSTRIDE];  // CLUSTER: this CTA's record, by column parity
  // PUSH: inbox[parity][source CTA][value] and one mbarrier per parity
  __shared__ __align__(16) double inbox[PUSH ? 2 : 1][PUSH ? 16 : 1][PSTRIDE];
  __shared__ __align__(8) uint64_t ibar[2];
  __shared__ double TB[NB][NB + 1];  // TB[r][c]: top-block row r, leaf column c
  __shared__ double wred[LEAF_THREADS / 32][PSTRIDE];
  __shared__ double tot[PSTRIDE];
  __shared__ double wv[NB];
  __shared__ double sc[4];  // tau, scal, beta, flag
  extern __shared__ double slab_s[];  // S * LEAF_THREADS rows x NB columns
  __shared__ __align__(16) double stage[CLUSTER ? 2 : LEAF_MAX_CTAS * PREC];  // grid leaf: the G partial records
  constexpr int SLD = S * LEAF_THREADS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  double* L0 = P + c0 + c0 * ldp;  // leaf top-left
  const i64 slab_rows = h - c0 - nb;
  const i64 per = (slab_rows + G - 1) / G;
  const i64 rb = nb + (i64)cta * per;
  i64 re = rb + per;
  if (re > nb + slab_rows) re = nb + slab_rows;

  double v[R > 0 ? R : 1][NB];
  if constexpr (R > 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const i64 r = rb + tid + (i64)k * LEAF_THREADS;
#pragma unroll
      for (int l = 0; l < NB; ++l) v[k][l] = (r < re && l < nb) ? L0[r + (i64)l * ldp] : 0.0;
    }
  }
  if constexpr (S > 0) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int sr = k * LEAF_THREADS + tid;
      const i64 r = rb + (i64)(R + k) * LEAF_THREADS + tid;
#pragma unroll 8
      for (int l = 0; l < NB; ++l) slab_s[sr + l * SLD] = (r < re && l < nb) ? L0[r + (i64)l * ldp] : 0.0;
    }
  }
  for (int e = tid; e < NB * NB; e += LEAF_THREADS) {
    const int r = e % NB, c = e / NB;
    TB[r][c] = (r < nb && c < nb) ? L0[r + (i64)c * ldp] : 0.0;
  }
  if constexpr (PUSH) {
    if (tid == 0) {
      mbar_init(smem_addr(&ibar[0]), 1);
      mbar_init(smem_addr(&ibar[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();  // every CTA's barriers exist before the first push
  }
  __syncthreads();

#ifdef RUTV_LEAF_PROF
  long long tp[8];
#define LEAF_T(i) tp[i] = clock64()
#else
#define LEAF_T(i)
#endif
  for (int jj = 0; jj < NB; jj += 1) {
    if (jj >= nb) break;
    LEAF_T(0);
    // ---------------- phase A: partial sums over this CTA's rows
    double acc[PSTRIDE];
#pragma unroll
    for (int l = 0; l < PSTRIDE; ++l) acc[l] = 0.0;
    if constexpr (R > 0) {
      switch (jj) {
#define RUTV_PA(J) \
  case J:          \
    leaf_partials<J, R>(v, acc); \
    break;
        RUTV_CASES32(RUTV_PA)
#undef RUTV_PA
      }
    } else {
      const double* xcol = L0 + (i64)jj * ldp;
      for (i64 r = rb + tid; r < re; r += LEAF_THREADS) {
        const double x = xcol[r];
        acc[0] = fma(x, x, acc[0]);
#pragma unroll
        for (int l = 0; l < NB; ++l)
          if (l > jj && l < nb) acc[1 + l] = fma(x, L0[r + (i64)l * ldp], acc[1 + l]);
      }
    }
    if constexpr (S > 0) {
      // shared-memory rows (zero beyond the slab: no bounds test)
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const int sr = k * LEAF_THREADS + tid;
        const double x = slab_s[sr + jj * SLD];
        acc[0] = fma(x, x, acc[0]);
#pragma unroll
        for (int l = 0; l < NB; ++l)
          if (l > jj) acc[1 + l] = fma(x, slab_s[sr + l * SLD], acc[1 + l]);
      }
    }
#pragma unroll
    {
      // warp reduction of the 32 dot products as a butterfly reduce-scatter:
      // at stride s every lane sends half of its 2s-value window to lane ^ s and
      // adds the other half, so after 16+8+4+2+1 = 31 shuffles lane L holds
      // the warp total of value L (vs 5 x 32 shuffles for 32 separate
      // all-reductions, which dominated the per-column latency in ncu:
      // leaf 218 -> 181 us at h = 16384)
      double* v32 = acc + 1;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const bool upper = (lane & st) != 0;
#pragma unroll
        for (int i = 0; i < st; ++i) {
          const double send = upper ? v32[i] : v32[i + st];
          const double keep = upper ? v32[i + st] : v32[i];
          v32[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
        }
      }
      double nrm = warp_sum(acc[0]);
      if (cta == 0) {
        // the top-block rows below the diagonal count once (CTA 0): warp w takes
        // rows jj+1+4w .. +4 and lane L the column-L dot, added to the warp's
        // butterfly result for value L (was one thread per row, 32 dependent
        // shared loads on warp 0 of CTA 0 -- on every CTA's critical path)
        double dl = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = jj + 1 + 4 * warp + i;
          if (r < nb) dl = fma(TB[r][jj], TB[r][lane], dl);
        }
        const double dn = __shfl_sync(0xffffffffu, dl, jj);  // column jj itself: the norm part
        if (lane > jj && lane < nb) v32[0] += dl;
        nrm += dn;
      }
      wred[warp][1 + lane] = v32[0];
      if (lane == 0) wred[warp][0] = nrm;
    }
    LEAF_T(1);
    __syncthreads();
    LEAF_T(2);
    if constexpr (PUSH) {
      // the record of this CTA into every CTA's inbox (slot cta), completing
      // 8 bytes per value on the receiver's barrier of this column's parity;
      // thread 0 arms its own barrier for the G x 33 values it will receive.
      // A CTA cannot push column jj+2 into a parity another CTA still reads:
      // it needs that CTA's column jj+1 record first, sent after the read.
      const int par = jj & 1;
      const uint32_t bar = smem_addr(&ibar[par]);
      if (tid == 0) mbar_expect_tx(bar, (uint32_t)(G * PSTRIDE * 8));
      if (tid < PSTRIDE) {
        double s2 = 0.0;
#pragma unroll
        for (int w = 0; w < LEAF_THREADS / 32; ++w) s2 += wred[w][tid];
        const uint32_t dst = smem_addr(&inbox[par][cta][tid]);
        for (int c = 0; c < G; ++c) st_async_f64(mapa_rank(dst, c), s2, mapa_rank(bar, c));
      }
      mbar_wait_cluster(bar, (uint32_t)((jj >> 1) & 1));
      if (tid < PSTRIDE) {
        double vals[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) vals[c] = c < G ? inbox[par][c][tid] : 0.0;
        double s3 = 0.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) s3 += vals[c];
        tot[tid] = s3;
      }
      __syncthreads();
    } else if constexpr (CLUSTER) {
      cg::cluster_group cl = cg::this_cluster();
      if (tid < PSTRIDE) {

        double s2 = 0.0;
#pragma unroll
        for (int w = 0; w < LEAF_THREADS / 32; ++w) s2 += wred[w][tid];
        mine[jj & 1][tid] = s2;
      }
      // one cluster barrier per column: a CTA writes the other parity's record
      // next, and cannot write this one again before every CTA has passed the
      // next barrier, i.e. finished reading it
      cl.sync();
      // thread e < 33 sums value e over the G records straight from the other
      // CTAs' shared memory (all G DSMEM loads in flight, then a fixed-order
      // sum: every CTA obtains bitwise identical totals)
      if (tid < PSTRIDE) {
        double vals[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) vals[c] = c < G ? *cl.map_shared_rank(&mine[jj & 1][tid], c) : 0.0;
        double s3 = 0.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) s3 += vals[c];
        tot[tid] = s3;
      }
      __syncthreads();
    } else {
      double* pj = partials + (size_t)(jj & 1) * G * PREC;
      if (tid < PSTRIDE) {
        double s2 = 0.0;
#pragma unroll
        for (int w = 0; w < LEAF_THREADS / 32; ++w) s2 += wred[w][tid];
        pj[(size_t)cta * PREC + tid] = s2;
      }
      cg::this_grid().sync();
      // ---------------- phase B: every CTA reduces the partials in the same
      // order: all threads pull the G x 33 records from L2 into shared memory
      // at once (cp.async, one L2 round trip, no registers), then thread
      // e < 33 sums value e over the CTAs in a fixed order
      // (16-byte cp.async.cg: L2 only -- the records of this parity were
      // rewritten since the last read, an L1 copy could be stale)
      for (int e = 2 * tid; e < G * PREC; e += 2 * LEAF_THREADS)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(stage + e)),
                     "l"(pj + e)
                     : "memory");
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      if (tid < PSTRIDE) {
        double s3 = 0.0;
        for (int c = 0; c < G; ++c) s3 += stage[c * PREC + tid];
        tot[tid] = s3;
      }
      __syncthreads();
    }
    LEAF_T(3);
    if (warp == 0) {
      // dlarfg (every lane, identical) and the w entries in one warp: one barrier
      // beta = -sign(alpha) hypot(alpha, ||x'||) as one square root of
      // alpha^2 + ||x'||^2 (the exchange already carries ||x'||^2; equal to
      // dlarfg's up to rounding, without sqrt -> hypot on the critical path)
      const double alpha = TB[jj][jj];
      double t0 = 0.0, s0 = 0.0, b0 = alpha;
      const bool act = tot[0] != 0.0;
      if (act) {
        b0 = -copysign(sqrt(fma(alpha, alpha, tot[0])), alpha);
        t0 = (b0 - alpha) / b0;
        s0 = 1.0 / (alpha - b0);
      }
      wv[lane] = (act && lane > jj && lane < nb) ? TB[jj][lane] + s0 * tot[1 + lane] : 0.0;
      if (lane == 0) {
        sc[0] = t0;
        sc[1] = s0;
        sc[2] = b0;
        sc[3] = act ? 1.0 : 0.0;
      }
    }
    __syncthreads();
    const double t = sc[0], scal = sc[1];
    const bool active = sc[3] != 0.0;
    if (active) {
      if constexpr (R > 0) {
        switch (jj) {
#define RUTV_UP(J) \
  case J:          \
    leaf_update<J, R>(v, scal, t, wv); \
    break;
          RUTV_CASES32(RUTV_UP)
#undef RUTV_UP
        }
      } else {
        double* xw = L0 + (i64)jj * ldp;
        for (i64 r = rb + tid; r < re; r += LEAF_THREADS) {
          const double vv = xw[r] * scal;
          xw[r] = vv;
          const double tv = t * vv;
#pragma unroll
          for (int l = 0; l < NB; ++l)
            if (l > jj && l < nb) L0[r + (i64)l * ldp] = fma(-tv, wv[l], L0[r + (i64)l * ldp]);
        }
      }
      if constexpr (S > 0) {
#pragma unroll
        for (int k = 0; k < S; ++k) {
          const int sr = k * LEAF_THREADS + tid;
          const double vv = slab_s[sr + jj * SLD] * scal;
          slab_s[sr + jj * SLD] = vv;
          const double tv = t * vv;
#pragma unroll
          for (int l = 0; l < NB; ++l)
            if (l > jj) slab_s[sr + l * SLD] = fma(-tv, wv[l], slab_s[sr + l * SLD]);
        }
      }
    }
    {
      // replicated top block: thread (row r = tid/8, columns 4(tid%8) .. +4),
      // the 8 threads of a row in one warp (was element-parallel with a
      // division per element and a separate barrier for the column scaling:
      // ~12 % of the leaf's stall samples, ncu source profile).  The pivot row
      // j has the implicit unit reflector entry; column j is scaled in place
      // once the row's 8 threads have read it (__syncwarp)
      const int r = tid >> 3, cq = (tid & 7) * 4;
      const bool row_on = active && r >= jj && r < nb;
      double vv = 0.0;
      if (row_on) {
        vv = (r == jj) ? 1.0 : TB[r][jj] * scal;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int l = cq + q;
          if (l > jj && l < nb) TB[r][l] = fma(-t * vv, wv[l], TB[r][l]);
        }
      }
      __syncwarp();
      if (row_on && cq == 0 && r > jj) TB[r][jj] = vv;
    }
    if (tid == 0) {
      // read again only after the loop (the next column touches rows > jj)
      TB[jj][jj] = sc[2];
      if (cta == 0) tau[c0 + jj] = t;
    }
    __syncthreads();
    LEAF_T(4);
    LEAF_T(5);
#ifdef RUTV_LEAF_PROF
    if (tid == 0 && cta == 0 && jj == 8 && c0 == 0)
      printf("leafprof G=%d h=%lld: A %lld sync1 %lld exch %lld scal+update %lld tail %lld total %lld cycles\n", G,
             (long long)h, tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[5] - tp[0]);
#endif
  }
  __syncthreads();  // the last column's TB writes before the write-back
  if constexpr (CLUSTER) cg::this_cluster().sync();  // no CTA exits while its record may still be read
  // the factored leaf into P and its explicit reflectors W (unit diagonal,
  // zeros above) into Wx(0:h, c0:c0+nb): the slab rows are the same values
  double* W0 = Wx + c0 + c0 * ldw;
  if constexpr (R > 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const i64 r = rb + tid + (i64)k * LEAF_THREADS;
      if (r < re) {
#pragma unroll
        for (int l = 0; l < NB; ++l)
          if (l < nb) {
            L0[r + (i64)l * ldp] = v[k][l];
            W0[r + (i64)l * ldw] = v[k][l];
          }
      }
    }
  }
  if constexpr (S > 0) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int sr = k * LEAF_THREADS + tid;
      const i64 r = rb + (i64)(R + k) * LEAF_THREADS + tid;
      if (r < re) {
#pragma unroll 8
        for (int l = 0; l < NB; ++l)
          if (l < nb) {
            const double x = slab_s[sr + l * SLD];
            L0[r + (i64)l * ldp] = x;
            W0[r + (i64)l * ldw] = x;
          }
      }
    }
  }
  if constexpr (R == 0) {
    // rows in L2: already in P; copy them to W
    for (i64 r = rb + tid; r < re; r += LEAF_THREADS)
      for (int l = 0; l < nb; ++l) W0[r + (i64)l * ldw] = L0[r + (i64)l * ldp];
  }
  if (cta == 0) {
    for (int e = tid; e < nb * nb; e += LEAF_THREADS) {
      const int r = e % nb, c = e / nb;
      L0[r + (i64)c * ldp] = TB[r][c];
      W0[r + (i64)c * ldw] = r > c ? TB[r][c] : (r == c ? 1.0 : 0.0);
    }
  }
  // rows 0 .. c0 of W's leaf columns are zero
  for (i64 e = (i64)cta * LEAF_THREADS + tid; e < c0 * nb; e += (i64)G * LEAF_THREADS)
    Wx[e % c0 + (c0 + e / c0) * ldw] = 0.0;
}

// T_LL by recursive doubling (blocks beyond wl stay zero): T = [T1, -T1 S12 T2;
// 0, T2] merges blocks of 1, 2, 4, 8, 16 reflectors (the compact-WY product
// rule, exactly the dlarft recurrence in exact arithmetic; 5 parallel levels
// instead of 32 sequential steps).  Ss = W_L^T W_L, Ts = diag(tau) on entry.
__device__ __forceinline__ void tll_doubling(double (*Ss)[NB + 1], double (*Ts)[NB + 1], double (*Mm)[NB + 1],
                                             int tid, int nthr) {
#pragma unroll
  for (int sz = 1; sz < NB; sz *= 2) {
    // Mm = S12 T22 for every pair (rows a.., cols a+sz..) ; T22 upper triangular
    for (int e = tid; e < (NB / 2) * sz; e += nthr) {
      const int pair = e / (sz * sz), rem = e % (sz * sz);
      const int a = pair * 2 * sz, r = a + rem % sz, c = a + sz + rem / sz;
      double acc = 0.0;
      for (int l = a + sz; l <= c; ++l) acc = fma(Ss[r][l], Ts[l][c], acc);
      Mm[r][c] = acc;
    }
    __syncthreads();
    // T12 = -T11 Mm ; T11 upper triangular
    for (int e = tid; e < (NB / 2) * sz; e += nthr) {
      const int pair = e / (sz * sz), rem = e % (sz * sz);
      const int a = pair * 2 * sz, r = a + rem % sz, c = a + sz + rem / sz;
      double acc = 0.0;
      for (int l = r; l < a + sz; ++l) acc = fma(Ts[r][l], Mm[l][c], acc);
      Ts[r][c] = -acc;
    }
    __syncthreads();
  }
}

// T(c0:c0+w, c0:c0+w) from S = W^T W (same block) and tau: T_jj = tau_j,
// T(0:j, j) = -tau_j T(0:j,0:j) S(0:j, j)   (dlarft, forward, columnwise).  One warp.
// The compact-WY factor of one leaf (replaces the larft warp kernel, the two
// T-merge GEMMs and the fill): with S = W^T W_L (column block L of W^T W, rows
// 0 .. c0+wl),
//   T_LL  by recursive doubling: T = [T1, -T1 S12 T2; 0, T2] merges blocks of
//         1, 2, 4, 8, 16 reflectors (the compact-WY product rule, exactly the
//         dlarft recurrence in exact arithmetic; 5 parallel levels instead of 32
//         sequential steps)
//   M1    = S(0:c0, L) T_LL
//   T(0:c0, L) = -T(0:c0, 0:c0) M1   (T upper triangular; CTA c takes rows
//         32c .. 32c+32 so the grid is ceil(c0/32) CTAs)
//   T(L, L) = T_LL, T(L, 0:c0) = 0   (CTA 0)
// Dynamic shared memory: M1 (c0 x NB, ld c0; columns >= wl zero).
__global__ void __launch_bounds__(256) t_block_kernel(const double* __restrict__ SL, i64 lds,
                                                      const double* __restrict__ tau, int c0, int wl,
                                                      double* __restrict__ T, i64 ldt) {
  extern __shared__ double M1[];
  __shared__ double Ts[NB][NB + 1];
  __shared__ double Ss[NB][NB + 1];
  __shared__ double Mm[NB][NB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    Ss[r][c] = (r < wl && c < wl) ? SL[c0 + r + (i64)c * lds] : 0.0;
    Ts[r][c] = (r == c && r < wl) ? tau[c0 + r] : 0.0;
  }
  __syncthreads();
  tll_doubling(Ss, Ts, Mm, tid, blockDim.x);
  // ---- M1(i, :) = S(i, 0:wl) T_LL for every row this CTA's product reads
  const int i0 = blockIdx.x * NB;
  for (int i = i0 + tid; i < c0; i += blockDim.x) {
    double srow[NB];
#pragma unroll
    for (int l = 0; l < NB; ++l) srow[l] = l < wl ? SL[i + (i64)l * lds] : 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l <= j; ++l) acc = fma(srow[l], Ts[l][j], acc);
      M1[i + j * c0] = acc;
    }
  }
  __syncthreads();
  // ---- T(i, c0 + j) = -sum_{l >= i} T(i, l) M1(l, j): warp w takes columns 4w .. 4w+4
  {
    const int lane = tid & 31, w = tid >> 5;
    const int i = i0 + lane;
    if (i < c0) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int l = i; l < c0; ++l) {
        const double til = T[i + (i64)l * ldt];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(til, M1[l + (4 * w + q) * c0], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * w + q < wl) T[i + (i64)(c0 + 4 * w + q) * ldt] = -acc[q];
    }
  }
  // ---- T(L, L) = T_LL, T(L, 0:c0) = 0
  if (blockIdx.x == 0)
    for (int e = tid; e < wl * (c0 + wl); e += blockDim.x) {
      const int r = e % wl, c = e / wl;
      T[c0 + r + (i64)c * ldt] = c < c0 ? 0.0 : Ts[r][c - c0];
    }
}


// ---------------------------------------------------------------- fused leaf update
// After qr_leaf_kernel has factored leaf L = columns [c0, c0+wl) of the h x w
// panel, ONE cooperative grid does what the S GEMM (+ split-K reduce),
// t_block_kernel and the three trailing GEMMs (+ reduce) did in 6-7 launches
// of ~25 us each (profiles/kernels_qr_r02.txt: 29 GEMM launches = 0.83 ms of a
// 16384 x 256 panel's 2.1 ms, latency not flops):
//   phase 1  each CTA c, rows R_c of [c0, h):  Q_c = W_L(R_c)^T X(R_c, 0:w),
//            X = [W(:, 0:c0+wl) | P(:, c0+wl:w)]   (NB x w partial, DMMA)
//   phase 2  Q = sum_c Q_c in a fixed order (CTA c reduces a slice)
//            -> S(0:c0+wl, L) = Q(:, 0:c0+wl)^T,  Z = W_L^T C = Q(:, c0+wl:w)
//   phase 3  T_LL from S_LL and tau (recursive doubling, every CTA);
//            T(0:c0, L) = -T(0:c0, 0:c0) S(0:c0, L) T_LL  (CTA c: rows 32c..);
//            C(R_c, :) -= W_L(R_c) (T_LL^T Z)   (C = P(c0:h, c0+wl:w), DMMA)
// Every CTA updates only its own rows, so phase 3 needs no further barrier.
// All sums are fixed-order: the factorisation stays bitwise reproducible for
// a given (h, w) (G depends on h - c0 and the SM count only).
constexpr int UPD_THREADS = 256;
constexpr int UPD_KC = 32;            // rows per staged chunk (= lanes: thread (lane, warp) stages row lane)
constexpr int UPD_NC = 128;           // X / C columns per pass (8 warps x 16)
constexpr int UPD_LD = UPD_KC + 4;    // staged chunk: column-major, padded
constexpr int UPD_ZLD = UPD_NC + 4;   // Z / M2 chunk: row-major (k, col), padded
constexpr int UPD_MAX_CTAS = 160;
constexpr int UPD_MIN_ROWS = 64;      // rows per CTA at least
static_assert(UPD_KC == 32 && UPD_NC == 128 && UPD_THREADS == 256, "panel_update_kernel's staging map");
constexpr size_t UPD_SMEM =
    sizeof(double) * ((size_t)NB * UPD_LD + (size_t)UPD_NC * UPD_LD + 2 * (size_t)NB * UPD_ZLD + 3 * NB * (NB + 1));

__device__ __forceinline__ void dmma884q(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(UPD_THREADS, 1)
    panel_update_kernel(double* __restrict__ P, i64 h, i64 ldp, const double* __restrict__ Wx, i64 ldw, i64 w,
                        i64 c0, int wl, const double* __restrict__ tau, double* __restrict__ T, i64 ldt,
                        double* __restrict__ rec, double* __restrict__ Qr) {
  extern __shared__ __align__(16) double usm[];
  double* Ws = usm;                              // W_L chunk: Ws[j * UPD_LD + kk] = W_L(r0 + kk, j)
  double* Xs = Ws + NB * UPD_LD;                 // X chunk:   Xs[c * UPD_LD + kk] = X(r0 + kk, n0 + c)
  double* Zs = Xs + UPD_NC * UPD_LD;             // Z chunk:   Zs[l * UPD_ZLD + c]
  double* M2 = Zs + NB * UPD_ZLD;                // T_LL^T Z:  M2[k * UPD_ZLD + c]
  double(*Ts)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(M2 + NB * UPD_ZLD);
  double(*Ss)[NB + 1] = Ts + NB;
  double(*Mm)[NB + 1] = Ss + NB;

  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int G = gridDim.x, cta = blockIdx.x;
  const i64 rows = h - c0;
  const i64 per = (rows + G - 1) / G;
  const i64 rb = c0 + (i64)cta * per;
  const i64 re = rb + per < h ? rb + per : h;  // rb >= re: no rows (zero record)
  const double* WL = Wx + c0 * ldw;             // column c0 of W, absolute rows
  const i64 E = (i64)NB * w;                    // entries of Q (NB x w, ld NB)

  // ---------------- phase 1: Q_c = W_L(R_c)^T X(R_c, :)
  // chunk loads double-buffered in registers: chunk k+1 is in flight while
  // chunk k's DMMAs run (one L2 round trip per pass, not per chunk)
  constexpr int XQ = UPD_NC * UPD_KC / UPD_THREADS, WQ = NB * UPD_KC / UPD_THREADS;
  for (i64 n0 = 0; n0 < w; n0 += UPD_NC) {
    double acc[4][2][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    // thread (lane, warp) stages row r0 + lane of columns warp + 8q: per-pass
    // column pointers, so a chunk load is one predicated load per element
    const double* xp[XQ];
#pragma unroll
    for (int q = 0; q < XQ; ++q) {
      const i64 col = n0 + warp + 8 * q;
      xp[q] = col >= w ? nullptr : (col < c0 + wl ? Wx + col * ldw : P + col * ldp);
    }
    const double* wp[WQ];
#pragma unroll
    for (int q = 0; q < WQ; ++q) wp[q] = warp + 8 * q < wl ? WL + (i64)(warp + 8 * q) * ldw : nullptr;
    double xv[XQ], wv[WQ];
    auto fetch = [&](i64 r0) {
      const i64 r = r0 + lane;
      const bool rin = r < re;
#pragma unroll
      for (int q = 0; q < XQ; ++q) xv[q] = (rin && xp[q]) ? xp[q][r] : 0.0;
#pragma unroll
      for (int q = 0; q < WQ; ++q) wv[q] = (rin && wp[q]) ? wp[q][r] : 0.0;
    };
    if (rb < re) fetch(rb);
    for (i64 r0 = rb; r0 < re; r0 += UPD_KC) {
      __syncthreads();  // the previous chunk is consumed
#pragma unroll
      for (int q = 0; q < XQ; ++q) Xs[(warp + 8 * q) * UPD_LD + lane] = xv[q];
#pragma unroll
      for (int q = 0; q < WQ; ++q) Ws[(warp + 8 * q) * UPD_LD + lane] = wv[q];
      __syncthreads();
      if (r0 + UPD_KC < re) fetch(r0 + UPD_KC);
#pragma unroll
      for (int kk = 0; kk < UPD_KC; kk += 4) {
        double a[4], b[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = Ws[(mi * 8 + g) * UPD_LD + kk + t];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) b[ni] = Xs[(warp * 16 + ni * 8 + g) * UPD_LD + kk + t];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma884q(acc[mi][ni], a[mi], b[ni]);
      }
    }
    // lane (g, t) holds Q_c(mi*8 + g, n0 + warp*16 + ni*8 + 2t + {0, 1})
    double* rc = rec + (i64)cta * E;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const i64 col = n0 + warp * 16 + ni * 8 + 2 * t + e;
          if (col < w) rc[(mi * 8 + g) + col * NB] = acc[mi][ni][e];
        }
  }
  grid.sync();

  // ---------------- phase 2: Q = sum_c Q_c (CTA c: entries [c*epc, (c+1)*epc);
  // four thread groups each load their <= UPD_MAX_CTAS/4 records at once, sum
  // them in record order, and the four sums are combined in a fixed order)
  {
    const i64 epc = (E + G - 1) / G;
    const i64 e0 = (i64)cta * epc, e1 = e0 + epc < E ? e0 + epc : E;
    const int grp = tid >> 6, gl = tid & 63;
    double* red = Zs;  // scratch
    for (i64 eb = e0; eb < e1; eb += 64) {
      const i64 e = eb + gl;
      double s = 0.0;
      if (e < e1) {
        constexpr int RQ = UPD_MAX_CTAS / 4;
        double x[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const int c = grp + 4 * q;
          x[q] = c < G ? __ldcg(rec + (i64)c * E + e) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < RQ; ++q) s += x[q];
      }
      __syncthreads();
      red[tid] = s;
      __syncthreads();
      if (grp == 0 && e < e1) Qr[e] = ((red[gl] + red[64 + gl]) + red[128 + gl]) + red[192 + gl];
    }
  }
  grid.sync();

  // ---------------- phase 3a: T_LL (every CTA)
  for (int e = tid; e < NB * NB; e += UPD_THREADS) {
    const int r = e % NB, c = e / NB;
    Ss[r][c] = (r < wl && c < wl) ? __ldcg(Qr + r + (c0 + c) * NB) : 0.0;
    Ts[r][c] = (r == c && r < wl) ? tau[c0 + r] : 0.0;
  }
  __syncthreads();
  tll_doubling(Ss, Ts, Mm, tid, UPD_THREADS);

  // ---------------- phase 3b: T(0:c0, L) = -T(0:c0, 0:c0) M1, M1 = S(0:c0, L) T_LL
  // (S(l, j) = Q(j, l)).  Row blocks of 32 from the LAST CTA down (the trailing
  // CTAs hold the fewest rows); per 32-column chunk l of T: the Q block and the
  // T block are staged in shared memory, M1's chunk formed there.
  for (i64 ib = G - 1 - cta; ib * NB < c0; ib += G) {
    const i64 i0 = ib * NB;
    double* Qc = Xs;            // Qc[m * NB + ll] = Q(m, lb + ll)   (NB x NB)
    double* Tc = Xs + NB * NB;  // Tc[ll * NB + ii] = T(i0 + ii, lb + ll)
    double at[4] = {0.0, 0.0, 0.0, 0.0};
    const int ii = lane;
    for (i64 lb = i0; lb < c0; lb += NB) {
      __syncthreads();
      for (int e = tid; e < NB * NB; e += UPD_THREADS) {
        const int m = e % NB, ll = e / NB;  // Q(:, lb + ll) is contiguous
        const i64 l = lb + ll;
        Qc[m * NB + ll] = l < c0 ? __ldcg(Qr + m + l * NB) : 0.0;
        const i64 i = i0 + m;  // here m plays the row ii of the T block
        Tc[ll * NB + m] = (l < c0 && i < c0 && l >= i) ? T[i + l * ldt] : 0.0;
      }
      __syncthreads();
      for (int e = tid; e < NB * NB; e += UPD_THREADS) {
        const int ll = e % NB, jj = e / NB;
        double a = 0.0;
        for (int m = 0; m <= jj; ++m) a = fma(Qc[m * NB + ll], Ts[m][jj], a);
        Mm[ll][jj] = a;
      }
      __syncthreads();
#pragma unroll 8
      for (int ll = 0; ll < NB; ++ll) {
        const double til = Tc[ll * NB + ii];
#pragma unroll
        for (int q = 0; q < 4; ++q) at[q] = fma(til, Mm[ll][4 * warp + q], at[q]);
      }
    }
    if (i0 + ii < c0)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * warp + q < wl) T[i0 + ii + (c0 + 4 * warp + q) * ldt] = -at[q];
  }
  // T(L, L) = T_LL, T(L, 0:c0) = 0
  if (cta == 0)
    for (i64 e = tid; e < (i64)wl * (c0 + wl); e += UPD_THREADS) {
      const i64 r = e % wl, c = e / wl;
      T[c0 + r + c * ldt] = c < c0 ? 0.0 : Ts[r][c - c0];
    }

  // ---------------- phase 3c: C(R_c, :) -= W_L(R_c) M2,  M2 = T_LL^T Z
  const i64 cb = c0 + wl, nrest = w - cb;
  for (i64 n0 = 0; n0 < nrest; n0 += UPD_NC) {
    __syncthreads();
    for (int e = tid; e < NB * UPD_NC; e += UPD_THREADS) {
      const int l = e % NB, c = e / NB;
      const i64 col = cb + n0 + c;
      Zs[l * UPD_ZLD + c] = (l < wl && col < w) ? __ldcg(Qr + l + col * NB) : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < NB * UPD_NC; e += UPD_THREADS) {
      const int c = e % UPD_NC, k = e / UPD_NC;
      double a = 0.0;
      for (int l = 0; l <= k; ++l) a = fma(Ts[l][k], Zs[l * UPD_ZLD + c], a);
      M2[k * UPD_ZLD + c] = a;
    }
    double wv[WQ], cv[4][2][2];
    const double* wp[WQ];
#pragma unroll
    for (int q = 0; q < WQ; ++q) wp[q] = warp + 8 * q < wl ? WL + (i64)(warp + 8 * q) * ldw : nullptr;
    double* cp[2];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const i64 col = cb + n0 + warp * 16 + ni * 8 + g;
      cp[ni] = col < w ? P + col * ldp : nullptr;
    }
    // W_L rows and this thread's C entries of one chunk (issued together: one
    // L2 round trip per chunk, the C read of chunk k+1 overlapping chunk k)
    auto fetch3 = [&](i64 r0) {
      const i64 r = r0 + lane;
#pragma unroll
      for (int q = 0; q < WQ; ++q) wv[q] = (r < re && wp[q]) ? wp[q][r] : 0.0;
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const i64 rr = r0 + mi * 8 + 2 * t + e;
            cv[mi][ni][e] = (cp[ni] && rr < re) ? cp[ni][rr] : 0.0;
          }
    };
    if (rb < re) fetch3(rb);
    for (i64 r0 = rb; r0 < re; r0 += UPD_KC) {
      __syncthreads();  // M2 written / the previous Ws consumed
#pragma unroll
      for (int q = 0; q < WQ; ++q) Ws[(warp + 8 * q) * UPD_LD + lane] = wv[q];
      __syncthreads();
      double acc[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < NB; kk += 4) {
        double a[4], b[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = Ws[(kk + t) * UPD_LD + mi * 8 + g];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) b[ni] = M2[(kk + t) * UPD_ZLD + warp * 16 + ni * 8 + g];
        // transposed tile: lane (g, t) gets (W_L M2)(rows 2t, 2t+1 of m-tile mi, column g of n-tile ni)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma884q(acc[mi][ni], b[ni], a[mi]);
      }
      double out[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) out[mi][ni][e] = cv[mi][ni][e] - acc[mi][ni][e];
      if (r0 + UPD_KC < re) fetch3(r0 + UPD_KC);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        if (cp[ni]) {
          double* pc = cp[ni];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const i64 r = r0 + mi * 8 + 2 * t + e;
              if (r < re) pc[r] = out[mi][ni][e];
            }
        }
      }
    }
  }
}

constexpr int kLeafClusterMax = 16;

// RUTV_LEAF_CLUSTER=0 forces the cooperative-grid leaf (tuning only)
bool leaf_cluster_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_LEAF_CLUSTER");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// Leaf grid: one thread-block cluster of <= 16 CTAs whenever the slab fits in
// its registers + shared memory (R rows per thread in registers, S in shared
// memory: up to 16 * 256 * 5 = 20480 rows); else a cooperative grid with R
// rows per thread in registers (R = 1, 2) or rows in L2 (R = 0).  G, R, S
// depend on the panel height only, so the factorisation is bitwise
// reproducible.
void leaf_plan(i64 slab_rows, int* G, int* R, int* S) {
  *S = 0;
  if (leaf_cluster_on()) {
    const i64 per_cta_rows = (i64)kLeafClusterMax * LEAF_THREADS;  // rows per (R + S) unit over 16 CTAs
    static int maxu = -1;  // RUTV_LEAF_MAXUNITS: cap on (R + S) rows per thread of the cluster leaf (tuning)
    if (maxu < 0) {
      const char* e = getenv("RUTV_LEAF_MAXUNITS");
      // measured (tools/leaf_ab.sh): the cluster leaf wins up to 3 rows per
      // thread (slab <= 12288); taller slabs are faster on the 64+ CTA grid
      maxu = e ? atoi(e) : 3;
    }
    for (int units = 1; units <= maxu; ++units) {
      if (slab_rows <= per_cta_rows * units) {
        const int r = units >= 2 ? 2 : 1;
        *R = r;
        *S = units - r;
        const i64 rows_per_cta = (i64)units * LEAF_THREADS;
        i64 g = (slab_rows + rows_per_cta - 1) / rows_per_cta;
        *G = (int)(g < 1 ? 1 : g);
        return;
      }
    }
  }
  const i64 cap1 = (i64)LEAF_MAX_CTAS * LEAF_THREADS;
  // RUTV_LEAF_R2_FROM: 2 rows per thread from this slab height on (grid
  // leaves).  Default: every grid leaf (slab > 12288) -- half the CTAs, so half
  // the partial records per column exchange (16384 rows: 145 -> 141 us; 20000:
  // 152 -> 144 us, tools/gpu_session.sh leaf_ab)
  static i64 r2_from = -2;
  if (r2_from == -2) {
    const char* e = getenv("RUTV_LEAF_R2_FROM");
    r2_from = e ? atoll(e) : 1;
  }
  i64 g;
  if (r2_from > 0 && slab_rows >= r2_from && slab_rows <= 2 * cap1) {
    *R = 2;
    g = (slab_rows + 2 * LEAF_THREADS - 1) / (2 * LEAF_THREADS);
  } else if (slab_rows <= cap1) {
    *R = 1;
    g = (slab_rows + LEAF_THREADS - 1) / LEAF_THREADS;
  } else if (slab_rows <= 2 * cap1) {
    *R = 2;
    g = (slab_rows + 2 * LEAF_THREADS - 1) / (2 * LEAF_THREADS);
  } else {
    *R = 0;
    g = LEAF_MAX_CTAS;
  }
  if (g < 1) g = 1;
  if (g > LEAF_MAX_CTAS) g = LEAF_MAX_CTAS;
  *G = (int)g;
}

// RUTV_LEAF_PUSH=0: the cluster-barrier + DSMEM-load exchange (A/B only)
bool leaf_push_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_LEAF_PUSH");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

template <int R, int S>
int launch_leaf_cluster(const Launch& L, int G, void** args) {
  void* fn = leaf_push_on() ? (void*)qr_leaf_kernel<R, true, S, true> : (void*)qr_leaf_kernel<R, true, S>;
  const size_t smem = (size_t)S * LEAF_THREADS * NB * sizeof(double);
  RUTV_ONCE_PER_DEVICE({
    RUTV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RUTV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(LEAF_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RUTV_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  return 0;
}

}  // namespace

// leaf records, then the fused update's per-CTA records and the reduced Q
i64 panel_qr_partials_elems(i64 h, i64 w) {
  (void)h;
  return LEAF_REC_ELEMS + (i64)(UPD_MAX_CTAS + 1) * NB * w;
}

namespace {
// RUTV_QR_FUSED=0 keeps the per-leaf S GEMM + t_block + trailing GEMMs (A/B only)
bool qr_fused_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_QR_FUSED");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

int launch_panel_update(const Launch& L, i64 h, i64 w, double* P, i64 ldp, const double* Wx, i64 ldw, i64 c0,
                        int wl, const double* tau, double* Tf, i64 ldtf, const QrWork& qw) {
  const i64 rows = h - c0;
  i64 G = (rows + UPD_MIN_ROWS - 1) / UPD_MIN_ROWS;
  const i64 gmax = L.device_sms < UPD_MAX_CTAS ? L.device_sms : UPD_MAX_CTAS;
  if (G > gmax) G = gmax;
  if (G < 1) G = 1;
  double* rec = qw.partials + LEAF_REC_ELEMS;
  double* Qr = rec + (i64)UPD_MAX_CTAS * NB * w;
  RUTV_ONCE_PER_DEVICE(RUTV_CUDA(
      cudaFuncSetAttribute(panel_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)UPD_SMEM)));
  double* Pp = P;
  const double* Wp = Wx;
  const double* tp = tau;
  double* Tp = Tf;
  i64 hh = h, lp = ldp, lw = ldw, ww = w, cc = c0, lt = ldtf;
  int wlv = wl;
  void* args[] = {&Pp, &hh, &lp, &Wp, &lw, &ww, &cc, &wlv, &tp, &Tp, &lt, &rec, &Qr};
  const size_t pe = L.pbegin();
  RUTV_CUDA(cudaLaunchCooperativeKernel((void*)panel_update_kernel, dim3((unsigned)G), dim3(UPD_THREADS), args,
                                        UPD_SMEM, L.stream));
  L.count();
  // algorithmic: Q (2 wl w rows) + the trailing update (2 rows wl nrest)
  L.pend(PK_DGEMM, 2.0 * (double)rows * wl * (double)(2 * w - c0 - wl), 8.0 * (double)rows * (w + wl + (w - c0 - wl)),
         pe, wl, w, rows);
  return 0;
}
}  // namespace

int panel_qr(const Launch& L, i64 h, i64 w, double* P, i64 ldp, double* tau, double* Wx, i64 ldw, double* Tf,
             i64 ldtf, const QrWork& qw) {
  if (w <= 0) return 0;
  if (h < w) return -2;
  for (i64 c0 = 0; c0 < w; c0 += NB) {
    const int wl = (int)((w - c0) < NB ? (w - c0) : NB);
    // ---- leaf factorisation (cooperative grid)
    {
      int G = 1, R = 1, S = 0;
      leaf_plan(h - c0 - wl, &G, &R, &S);
      double* Pp = P;
      i64 hh = h, ld = ldp, cc = c0;
      int nbv = wl;
      double* taup = tau;
      double* part = qw.partials;
      double* wxp = Wx;
      i64 ldwv = ldw;
      void* args[] = {&Pp, &hh, &ld, &cc, &nbv, &taup, &part, &wxp, &ldwv};
      const size_t pe = L.pbegin();
      if (G <= kLeafClusterMax && R > 0 && leaf_cluster_on()) {
        // one thread-block cluster of G CTAs (non-portable size up to 16)
        const int units = R + S;
        if (units == 1) RUTV_TRY((launch_leaf_cluster<1, 0>(L, G, args)));
        else if (units == 2) RUTV_TRY((launch_leaf_cluster<2, 0>(L, G, args)));
        else if (units == 3) RUTV_TRY((launch_leaf_cluster<2, 1>(L, G, args)));
        else if (units == 4) RUTV_TRY((launch_leaf_cluster<2, 2>(L, G, args)));
        else RUTV_TRY((launch_leaf_cluster<2, 3>(L, G, args)));
      } else {
        void* fn = R == 1 ? (void*)qr_leaf_kernel<1, false>
                          : (R == 2 ? (void*)qr_leaf_kernel<2, false> : (void*)qr_leaf_kernel<0, false>);
        RUTV_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(LEAF_THREADS), args, 0, L.stream));
      }
      L.count();
      // algorithmic: ~4 (h-c0) wl^2 flops (dlarfg + dlarf over the leaf); bytes: the leaf read + written once
      L.pend(PK_QR_LEAF, 4.0 * (double)(h - c0) * wl * wl, 16.0 * (double)(h - c0) * wl, pe);
    }
    // (the leaf kernel wrote the explicit W of this leaf)
    if (qr_fused_on() && qw.partials_elems >= panel_qr_partials_elems(h, w)) {
      RUTV_TRY(launch_panel_update(L, h, w, P, ldp, Wx, ldw, c0, wl, tau, Tf, ldtf, qw));
      continue;
    }
    // ---- S(0:c0+wl, L) = W(c0:h, 0:c0+wl)^T W(c0:h, L)
    double* SL = qw.S + c0 * w;  // S stored w x w, ld w
    RUTV_TRY(launch_dgemm(L, true, false, c0 + wl, wl, h - c0, 1.0, Wx + c0, ldw, Wx + c0 + c0 * ldw, ldw, 0.0,
                          SL, w, qw.gemm_ws, qw.gemm_ws_elems));
    // ---- T(:, L): T_LL, T(0:c0, L) = -T(0:c0,0:c0) S(0:c0,L) T_LL, T(L, 0:c0) = 0
    {
      const size_t smem = (size_t)(c0 > 0 ? c0 : 1) * NB * sizeof(double);
      // up to c0 = 640 (b = 672) with the 17 KB of static shared memory
      RUTV_ONCE_PER_DEVICE(
          RUTV_CUDA(cudaFuncSetAttribute(t_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024)));
      if (smem > 160 * 1024) return -3;
      const int tb = c0 > 0 ? (int)((c0 + NB - 1) / NB) : 1;
      t_block_kernel<<<tb, 256, smem, L.stream>>>(SL, w, tau, (int)c0, wl, Tf, ldtf);
      L.count();
      RUTV_CHECK_LAUNCH("t_block_kernel");
    }
    // ---- trailing panel update C -= W_L T_LL^T (W_L^T C), C = P(c0:h, c0+wl:w)
    const i64 nrest = w - c0 - wl;
    if (nrest > 0) {
      double* Cp = P + c0 + (c0 + wl) * ldp;
      const double* WL = Wx + c0 + c0 * ldw;
      RUTV_TRY(launch_dgemm(L, true, false, wl, nrest, h - c0, 1.0, WL, ldw, Cp, ldp, 0.0, qw.tmp3, wl,
                            qw.gemm_ws, qw.gemm_ws_elems));
      RUTV_TRY(launch_dgemm(L, true, false, wl, nrest, wl, 1.0, Tf + c0 + c0 * ldtf, ldtf, qw.tmp3, wl, 0.0,
                            qw.tmp2, wl, nullptr, 0));
      RUTV_TRY(launch_dgemm(L, false, false, h - c0, nrest, wl, -1.0, WL, ldw, qw.tmp2, wl, 1.0, Cp, ldp, nullptr,
                            0));
    }
  }
  return 0;
}

}  // namespace rutv
