// K2 -- the FP64 dense contractions of randUTV on the B200 tensor cores.
//
// Every flop-heavy step of the loop is a product of column blocks:
//   S2/S3  Y = A_t^T G,  Z = A_t Y,  Y = A_t^T Z
//   S5     Z = X W_V,  X -= (Z T_V) W_V^T  for X = T, V
//   S7     Z = W_U^T X,  X -= W_U (T_U^T Z);  U likewise
//   S9     the SVD folds A01 V_SVD, U_SVD^T A12, U1 U_SVD, V1 V_SVD
// so one GEMM kernel C = alpha op(A) op(B) + beta C serves them all.
//
// sm_100a has no FP64 kind of tcgen05.mma (ptxas rejects .kind::f64), so FP64
// tensor work is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); the
// measured chip peak is 37.0 TFLOP/s (profiles/fp64_peak_r01.json), equal to
// the DFMA peak, and DMMA needs 8x fewer issue slots.  Design (each choice
// measured on B200, profiles/gemm_tuning_r01.txt):
//   * CTA tile 64 x 64, BK = 32, 128 threads = 4 warps (2 x 2) of 32 x 32
//     (4 x 4 DMMA tiles, 32 accumulators/thread), 2 cp.async stages (36.9 KB
//     each), 3 CTAs per SM.  Round 2: BK 16 -> 32 with 3 -> 2 stages (the same
//     32-deep prefetch, half the k-tile barriers per DMMA) took the large c3
//     shapes from 33.6 to 34.5 TFLOP/s and the c3 step +1.7 %
//     (profiles/gemm_ab_r02.txt); cuBLAS's d884 kernel: 35.5-35.8.
//   * Shared layout follows the global contiguous dimension with a 4-double row
//     pad (conflict-free 64-bit fragment loads); fragments double-buffered in
//     registers; one wait + barrier per k-tile, placed before the last k-step.
//   * Interior tiles copy with a bounds-free cp.async path (per-item chunk
//     pointers, ~3 instructions per 16-byte copy): the general masked path
//     cost ~25 integer instructions per copy and capped the kernel at ~80 %.
//   * Persistent grid with a dynamic tile scheduler (per-stream atomic
//     counter) and a cp.async ring flattened over (item, k-tile), so the next
//     item's loads overlap the current item's epilogue; the DMMA computes the
//     transposed 8x8 tile so each lane owns two consecutive rows of C
//     (16-byte epilogue accesses); read-modify-write epilogues prefetch their C
//     tile into L2 a few k-tiles ahead.
//   * Skinny outputs with long K (A_t^T G, W^T X: K up to 262144) split K by a
//     wave-quantisation time model; partial tiles go to a workspace and a
//     second kernel sums them in a fixed order, so results are bitwise
//     deterministic run to run.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace rutv {

namespace {

#ifndef RUTV_GEMM_BK  // k-tile depth (A/B tuning override; the default is the measured best)
#define RUTV_GEMM_BK 32
#endif
constexpr int BK = RUTV_GEMM_BK;
// Shared-memory tile layout.  A tile is Lo rows of Lc doubles (Lc along the
// operand's contiguous global dimension).  The 8-byte fragment loads of a
// half-warp hit rows o..o+3 at the same column offsets, so a plain layout has
// 4-way bank conflicts.  RUTV_GEMM_SWZ = 0 (default): rows padded to Lc + 4
// doubles; 1: element (o, c) lives at o*Lc + (c ^ 4*(o & 3)) -- also
// conflict-free, no padding (16 KB per 64x64x16 stage, so 4 stages fit 3
// CTAs/SM), measured 1 % slower on B200 with 4 stages (profiles/gemm_tuning_r01.txt).
#ifndef RUTV_GEMM_SWZ
#define RUTV_GEMM_SWZ 0
#endif
constexpr int PAD = RUTV_GEMM_SWZ ? 0 : 4;
__host__ __device__ constexpr int soff(int o, int c, int Lc) {
  return RUTV_GEMM_SWZ ? o * Lc + (c ^ ((o & 3) << 2)) : o * (Lc + PAD) + c;
}

// Tile configuration: BM x BN CTA tile, WM x (NW/WM) warps, STAGES-deep ring,
// MINB CTAs per SM.
template <int BM_, int BN_, int WM_, int STAGES_, int MINB_, int NW_ = 8>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = NW_ / WM_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = 32 * NW_;
  static constexpr int MI = BM / (WM * 8), NI = BN / (WN * 8);
  static constexpr int A_ELEMS = (BK * (BM + PAD) > BM * (BK + PAD)) ? BK * (BM + PAD) : BM * (BK + PAD);
  static constexpr int B_ELEMS = (BK * (BN + PAD) > BN * (BK + PAD)) ? BK * (BN + PAD) : BN * (BK + PAD);
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_ELEMS * sizeof(double);
};
//   Cfg< 64, 64,2,2,3,4>: 4 warps (2 x 2) of 32 x 32, 2 stages of BK = 32, 3 CTAs/SM (the
//                       CUTLASS d884 64x64 tile cuBLAS picks on B200, with a deeper k-tile)
#ifndef RUTV_GEMM_STAGES  // tuning overrides (tools/ab.sh); the defaults are the measured best
#define RUTV_GEMM_STAGES 2
#endif
#ifndef RUTV_GEMM_MINB
#define RUTV_GEMM_MINB 3
#endif
#ifndef RUTV_SPLIT_FIXED_US  // fixed cost of a split-K reduction launch in the split model (us)
#define RUTV_SPLIT_FIXED_US 12.0
#endif
#ifndef RUTV_RASTER_GROUP
#define RUTV_RASTER_GROUP 64
#endif
using CfgSmall = Cfg<64, 64, 2, RUTV_GEMM_STAGES, RUTV_GEMM_MINB, 4>;
//   Cfg<128, 64,2,3,2,4>: 4 warps (2 x 2) of 64 x 32 -- 32 independent DMMAs per warp and
//                       k-step instead of 16 (fewer fixed-latency stalls per DMMA), 2 CTAs/SM
using CfgWide = Cfg<128, 64, 2, RUTV_GEMM_STAGES, 2, 4>;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int VEC>
__device__ __forceinline__ void cp_async(uint32_t dst, const double* src, int src_bytes) {
  if constexpr (VEC == 2) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Copy one Lc x Lo tile (Lc along the global contiguous dimension) into shared
// memory (layout soff).  lim_c / lim_o: first invalid global index.
template <int Lc, int Lo, int VEC, int THREADS>
__device__ __forceinline__ void load_tile(double* sm, const double* __restrict__ g, i64 ld, i64 c0, i64 o0,
                                          i64 lim_c, i64 lim_o, int tid) {
  constexpr int CPR = Lc / VEC;           // chunks per row
  constexpr int NCH = CPR * Lo;           // chunks per tile
  static_assert(NCH % THREADS == 0, "tile/threads mismatch");
#pragma unroll
  for (int it = 0; it < NCH / THREADS; ++it) {
    const int ch = tid + it * THREADS;
    const int o = ch / CPR;
    const int ci = (ch % CPR) * VEC;
    const i64 gc = c0 + ci, go = o0 + o;
    i64 nvalid = lim_c - gc;
    nvalid = nvalid < 0 ? 0 : (nvalid > VEC ? VEC : nvalid);
    if (go >= lim_o) nvalid = 0;
    const double* src = nvalid > 0 ? g + gc + go * ld : g;
    cp_async<VEC>(smem_u32(sm + soff(o, ci, Lc)), src, (int)(nvalid * 8));
  }
}

// Interior fast path of load_tile: `g` is this thread's first chunk source,
// successive chunks are `gstep` elements apart, no bounds checks (the caller
// guarantees the tile and the k-tile are fully inside the operand).  ~3
// instructions per cp.async instead of ~25 for the general path.
template <int Lc, int Lo, int VEC, int THREADS>
__device__ __forceinline__ void load_tile_fast(double* sm, const double* __restrict__ g, i64 gstep, int tid) {
  constexpr int CPR = Lc / VEC, RPI = THREADS / CPR, NIT = CPR * Lo / THREADS;
  static_assert(THREADS % CPR == 0 && (CPR * Lo) % THREADS == 0, "tile/threads mismatch");
  const int o = tid / CPR, ci = (tid % CPR) * VEC;
#pragma unroll
  for (int it = 0; it < NIT; ++it) cp_async<VEC>(smem_u32(sm + soff(o + it * RPI, ci, Lc)), g + it * gstep, VEC * 8);
}

// this thread's first chunk within an Lc x Lo tile whose origin is (c0, o0)
template <int Lc, int VEC, int THREADS>
__device__ __forceinline__ const double* chunk0(const double* g, i64 ld, i64 c0, i64 o0, int tid) {
  constexpr int CPR = Lc / VEC;
  return g + (c0 + (tid % CPR) * VEC) + (o0 + tid / CPR) * ld;
}

// Persistent tile loop over the work items (whole tiles, then the k-ranges of
// the split tail tiles: see dgemm_kernel; consecutive items share a panel in
// L2, tile_origin).  Items differ in length (k-tiles), so the long ones come
// first.  With `sched` (two device ints, zero between launches) the
// CTAs claim items dynamically with atomicAdd -- CTAs that become resident late
// (e.g. while the side stream's Jacobi SVD holds SMs) simply take fewer items,
// so the grid never waits on a straggler; the last CTA to finish re-zeroes the
// counters for the next launch on the stream.  Without it, CTA c takes items
// c, c + gridDim.x, ...  The cp.async ring runs over the flattened sequence of
// (item, k-tile) iterations, so the next item's first k-tiles are loading
// while the current item's epilogue (C read-modify-write) runs.
constexpr int RING = 8;           // in-flight item ids (>= STAGES + 1)
constexpr int RASTER_GROUP = RUTV_RASTER_GROUP;  // tile rows per raster group

// Origin (in tiles) of output tile `tile` of a gm x gn tile grid.
__device__ __forceinline__ void tile_origin(int tile, int gm, int gn, int& tm, int& tn) {
  if (gn <= RASTER_GROUP / 2 || gm <= RASTER_GROUP / 2) {
    // skinny output: raster along the short side, so the few tiles sharing a
    // panel of the long operand run together (skinny A_t^T G: the 4 N-tiles of
    // an A_t panel read it from DRAM once instead of four times)
    if (gn <= gm) {
      tm = tile / gn;
      tn = tile % gn;
    } else {
      tm = tile % gm;
      tn = tile / gm;
    }
  } else {
    // grouped raster: groups of RASTER_GROUP tile rows walked column by
    // column, so the resident items share a few B panels and the group's A
    // panels stay in L2 while C streams through (a plain row-major raster
    // re-read the B operand of the c3 rank-2b update ~38x from DRAM: ncu,
    // 1.58x the compulsory bytes)
    const int g = tile / (RASTER_GROUP * gn), loc = tile % (RASTER_GROUP * gn);
    const int gr = (gm - g * RASTER_GROUP) < RASTER_GROUP ? gm - g * RASTER_GROUP : RASTER_GROUP;
    tm = g * RASTER_GROUP + loc % gr;
    tn = loc / gr;
  }
}

// Work items (tail-split schedule).  Items 0 .. full-1 are whole tiles
// 0 .. full-1 over all of K, written straight to C.  The remaining
// tail = tiles - full tiles are split into `tsplits` k-ranges of `kchunk`
// (item full + z*tail + tt: tile full + tt, k-range z); their partial tiles go
// to `part` in a compact layout (BM x BN column-major per (z, tt), at
// (z*tail + tt)*BM*BN) and tail_reduce_kernel sums them in the fixed order
// z = 0 .. tsplits-1.  full = tiles is the unsplit GEMM, full = 0 is plain
// split-K over every tile; a tail of the last partial wave split across the
// whole chip is the data-parallel + stream-K hybrid (the full waves run at
// full efficiency, only the ragged last wave is split).
template <class CF, bool TA, bool TB, int VA, int VB, bool CPF>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
    dgemm_kernel(i64 M, i64 N, i64 K, double alpha, const double* __restrict__ A, i64 lda,
                 const double* __restrict__ B, i64 ldb, double beta, double* __restrict__ C, i64 ldc,
                 i64 kchunk, int full, int tsplits, double* __restrict__ part, int* __restrict__ sched) {
  constexpr int BM = CF::BM, BN = CF::BN, STAGES = CF::STAGES, MI = CF::MI, NI = CF::NI;
  constexpr int A_ELEMS = CF::A_ELEMS, STAGE_ELEMS = CF::STAGE_ELEMS;
  extern __shared__ __align__(16) double smem[];
  __shared__ int ring[RING];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % CF::WM, wn = warp / CF::WM;
  const int gm = (int)((M + BM - 1) / BM), gn = (int)((N + BN - 1) / BN);
  const int tiles = gm * gn, tail = tiles - full, items = full + tail * tsplits;
  const int ktiles_full = (int)((K + BK - 1) / BK);

  // item id of sequence number `seq` of this CTA (thread 0 only)
  auto claim = [&](int seq) -> int {
    if (sched) return atomicAdd(sched, 1);
    return (int)blockIdx.x + seq * (int)gridDim.x;
  };
  struct TileP {
    i64 m0, n0, kb, ke;
    int slot;  // -1: whole tile, written to C; else partial slot z*tail + tt
    int nkt;
  };
  // per-item constants (the only integer divisions: once per item, 32-bit)
  auto params = [&](int item) {
    TileP tp;
    int tile;
    if (CPF || item < full) {  // the CPF instantiation runs unsplit GEMMs only
      tile = item;
      tp.slot = -1;
      tp.kb = 0;
      tp.ke = K;
      tp.nkt = ktiles_full;
    } else {
      const int j = item - full, z = j / tail;
      tile = full + (j - z * tail);
      tp.slot = j;
      tp.kb = (i64)z * kchunk;
      tp.ke = (tp.kb + kchunk < K) ? tp.kb + kchunk : K;
      tp.nkt = (int)((tp.ke - tp.kb + BK - 1) / BK);
    }
    int tm, tn;
    tile_origin(tile, gm, gn, tm, tn);
    tp.m0 = (i64)tm * BM;
    tp.n0 = (i64)tn * BN;
    return tp;
  };
  auto nkt_of = [&](const TileP& tp) { return CPF ? ktiles_full : tp.nkt; };
  // producer-side per-item constants of the fast path: the thread's first chunk
  // at k-tile 0 of each operand, and whether the tile is interior in M / N
  constexpr int THR = CF::THREADS;
  constexpr int RPI_A = THR / ((TA ? BK : BM) / VA), RPI_B = THR / ((TB ? BN : BK) / VB);
  const i64 gstepA = (i64)RPI_A * lda, gstepB = (i64)RPI_B * ldb;
  const i64 kstepA = TA ? (i64)BK : (i64)BK * lda, kstepB = TB ? (i64)BK * ldb : (i64)BK;
  const double* pa0 = A;
  const double* pb0 = B;
  bool p_inner = false;
  auto producer_item = [&](const TileP& tp) {
    pa0 = TA ? chunk0<BK, VA, THR>(A, lda, tp.kb, tp.m0, tid) : chunk0<BM, VA, THR>(A, lda, tp.m0, tp.kb, tid);
    pb0 = TB ? chunk0<BN, VB, THR>(B, ldb, tp.n0, tp.kb, tid) : chunk0<BK, VB, THR>(B, ldb, tp.kb, tp.n0, tid);
    p_inner = tp.m0 + BM <= M && tp.n0 + BN <= N;
  };
  auto load_stage = [&](int stage, const TileP& tp, int kt) {
    double* As = smem + stage * STAGE_ELEMS;
    double* Bs = As + A_ELEMS;
    const i64 k0 = tp.kb + (i64)kt * BK;
    if (p_inner && k0 + BK <= tp.ke) {
      if constexpr (!TA) load_tile_fast<BM, BK, VA, THR>(As, pa0 + kt * kstepA, gstepA, tid);
      else load_tile_fast<BK, BM, VA, THR>(As, pa0 + kt * kstepA, gstepA, tid);
      if constexpr (!TB) load_tile_fast<BK, BN, VB, THR>(Bs, pb0 + kt * kstepB, gstepB, tid);
      else load_tile_fast<BN, BK, VB, THR>(Bs, pb0 + kt * kstepB, gstepB, tid);
      return;
    }
    if constexpr (!TA) load_tile<BM, BK, VA, THR>(As, A, lda, tp.m0, k0, M, tp.ke, tid);   // rows: k, contiguous m
    else load_tile<BK, BM, VA, THR>(As, A, lda, k0, tp.m0, tp.ke, M, tid);                 // rows: m, contiguous k
    if constexpr (!TB) load_tile<BK, BN, VB, THR>(Bs, B, ldb, k0, tp.n0, tp.ke, N, tid);   // rows: n, contiguous k
    else load_tile<BN, BK, VB, THR>(Bs, B, ldb, tp.n0, k0, N, tp.ke, tid);                 // rows: k, contiguous n
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // epilogue of one item.  The DMMA computes the TRANSPOSED 8x8 tile (the
  // N-side fragment is fed as the mma's A operand), so lane (g, t) holds
  // C[rows 2t, 2t+1][col g]: two consecutive rows of one column, i.e. one
  // 16-byte load/store in column-major C (half the epilogue instructions).
  const bool cvec = (((uintptr_t)C & 15) == 0) && ((ldc & 1) == 0);
  auto epilogue = [&](const TileP& tp) {
    if (!CPF && tp.slot >= 0) {
      // partial tile of a k-range: compact BM x BN column-major slot, always
      // whole (the reduction reads only the in-range elements)
      double* pb = part + (i64)tp.slot * (BM * BN) + (wm * (MI * 8) + 2 * t) +
                   (wn * (NI * 8) + g) * BM;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          *reinterpret_cast<double2*>(pb + mi * 8 + ni * 8 * BM) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
          acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
      }
      return;
    }
    if (cvec && tp.m0 + BM <= M && tp.n0 + BN <= N) {
      // interior tile: no bounds checks, one base pointer, 16-byte accesses
      double* cb = C + (tp.m0 + wm * (MI * 8) + 2 * t) + (tp.n0 + wn * (NI * 8) + g) * ldc;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          double2* cp = reinterpret_cast<double2*>(cb + mi * 8 + (i64)(ni * 8) * ldc);
          double2 v;
          if (beta == 0.0) {
            v.x = alpha * acc[mi][ni][0];
            v.y = alpha * acc[mi][ni][1];
          } else {
            const double2 c = *cp;
            v.x = alpha * acc[mi][ni][0] + beta * c.x;
            v.y = alpha * acc[mi][ni][1] + beta * c.y;
          }
          *cp = v;
          acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
      }
      return;
    }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const i64 row = tp.m0 + wm * (MI * 8) + mi * 8 + 2 * t;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const i64 col = tp.n0 + wn * (NI * 8) + ni * 8 + g;
        double* cp = C + row + col * ldc;
        if (col < N) {
          if (cvec && row + 1 < M) {
            double2 v;
            if (beta == 0.0) {
              v.x = alpha * acc[mi][ni][0];
              v.y = alpha * acc[mi][ni][1];
            } else {
              const double2 c = *reinterpret_cast<const double2*>(cp);
              v.x = alpha * acc[mi][ni][0] + beta * c.x;
              v.y = alpha * acc[mi][ni][1] + beta * c.y;
            }
            *reinterpret_cast<double2*>(cp) = v;
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if (row + e < M) {
                cp[e] = (beta == 0.0) ? alpha * acc[mi][ni][e] : alpha * acc[mi][ni][e] + beta * cp[e];
              }
            }
          }
        }
        acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
    }
  };

  if (ktiles_full == 0) {  // K == 0: C = beta C (the host passes full = tiles)
    for (int w = blockIdx.x; w < items; w += gridDim.x) epilogue(params(w));
    return;
  }

  // ---- prologue: claim the items of the first STAGES-1 loads (no more: a
  // claimed item waits for this CTA even when others are idle)
  int min_nkt = full > 0 ? ktiles_full : (1 << 30);
  if (tail > 0) {
    const int c0 = (int)((kchunk + BK - 1) / BK), cl = (int)((K - (i64)(tsplits - 1) * kchunk + BK - 1) / BK);
    min_nkt = min(min_nkt, min(c0, cl));
  }
  const int pre = (STAGES - 1) / min_nkt + 1;
  if (tid == 0)
    for (int q = 0; q < pre; ++q) ring[q % RING] = claim(q);
  int claimed = pre;
  __syncthreads();
  int p_seq = 0, p_kt = 0, p_stage = 0;  // producer: next (item, k-tile, stage) to load
  int p_item = ring[0];
  bool p_need = false;
  TileP ptp = params(p_item < items ? p_item : 0);
  producer_item(ptp);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (p_item < items) load_stage(p_stage, ptp, p_kt);
    cp_async_commit();
    p_stage = p_stage + 1 == STAGES ? 0 : p_stage + 1;
    if (++p_kt == nkt_of(ptp)) {
      p_kt = 0;
      ++p_seq;
      p_item = ring[p_seq % RING];
      if (p_item < items) {
        ptp = params(p_item);
        producer_item(ptp);
      }
    }
  }

  // fragments of one k-step (4 of K), double-buffered in registers: the loads
  // for step kk+1 are issued before the DMMAs of step kk, and the per-k-tile
  // wait + barrier sits before the LAST step's DMMAs (whose fragments are
  // already in registers), so the barrier overlaps the DMMA pipe's backlog
  auto load_frags = [&](double (&a)[MI], double (&b)[NI], int stage, int kk) {
    const double* As = smem + stage * STAGE_ELEMS;
    const double* Bs = As + A_ELEMS;
    const int k = kk * 4 + t;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int row = wm * (MI * 8) + mi * 8 + g;
      a[mi] = TA ? As[soff(row, k, BK)] : As[soff(k, row, BM)];
    }
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int col = wn * (NI * 8) + ni * 8 + g;
      b[ni] = TB ? Bs[soff(k, col, BN)] : Bs[soff(col, k, BK)];
    }
  };
  // ---- main loop over the flattened (item, k-tile) sequence
  int c_seq = 0, c_kt = 0, c_stage = 0;  // consumer
  int c_item = ring[0];
  TileP ctp = params(c_item < items ? c_item : 0);
  double fa[2][MI], fb[2][NI];
  cp_async_wait<STAGES - 2>();
  __syncthreads();
  load_frags(fa[0], fb[0], 0, 0);
  while (c_item < items) {
    {  // producer: the copies of stage it + STAGES - 1 (last read in iteration it - 1,
       // before that iteration's barrier)
      if (p_need) {  // claimed in the previous iteration, published by its barrier
        p_item = ring[p_seq % RING];
        if (p_item < items) {
          ptp = params(p_item);
          producer_item(ptp);
        }
        p_need = false;
      }
      if (p_item < items) load_stage(p_stage, ptp, p_kt);
      cp_async_commit();
      p_stage = p_stage + 1 == STAGES ? 0 : p_stage + 1;
      if (++p_kt == nkt_of(ptp)) {
        p_kt = 0;
        ++p_seq;
        p_need = true;
        if (p_seq >= claimed) {
          if (tid == 0) ring[p_seq % RING] = (p_item < items) ? claim(p_seq) : items;
          claimed = p_seq + 1;
        }
      }
    }
    const int n_stage = c_stage + 1 == STAGES ? 0 : c_stage + 1;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      if (kk == BK / 4 - 1) {
        cp_async_wait<STAGES - 2>();  // stage n_stage has landed (this thread's copies) ...
        __syncthreads();              // ... and everyone's
        load_frags(fa[0], fb[0], n_stage, 0);
      } else {
        load_frags(fa[(kk + 1) & 1], fb[(kk + 1) & 1], c_stage, kk + 1);
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma884(acc[mi][ni], fb[kk & 1][ni], fa[kk & 1][mi]);  // transposed tile
    }
    c_stage = n_stage;
    // the epilogue's C read is latency-bound (ncu: its DFMAs carried ~25 % of the
    // stall samples): pull the item's C tile into L2 a few k-tiles ahead
    // (a separate instantiation: the branch alone costs the long-K products ~15 %)
    // (k-tile nkt - 3 of a whole tile: its C is read by the epilogue)
    if constexpr (CPF) if (c_kt == (ktiles_full > 3 ? ktiles_full - 3 : 0)) {
#pragma unroll
      for (int h = 0; h < (BM / 16) * BN / CF::THREADS; ++h) {
        const int line = tid + h * CF::THREADS;           // 128-byte lines: BM/16 per column
        const int cc = line / (BM / 16), rr = (line % (BM / 16)) * 16;
        const i64 row = ctp.m0 + rr, col = ctp.n0 + cc;
        if (row < M && col < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + row + col * ldc));
      }
    }
    if (++c_kt == nkt_of(ctp)) {
      epilogue(ctp);
      c_kt = 0;
      ++c_seq;
      c_item = ring[c_seq % RING];  // claimed before the producer needed it
      if (c_item < items) ctp = params(c_item);
    }
  }
  cp_async_wait<0>();
  if (sched) {
    __syncthreads();
    if (tid == 0) {
      // every claim of this launch happened-before this CTA's arrival
      __threadfence();
      if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
        sched[0] = 0;
        sched[1] = 0;
        __threadfence();
      }
    }
  }
}

// C(tail tiles) = alpha * sum_z part(z, tt) + beta C, z = 0 .. tsplits-1 in
// order (bitwise deterministic).  Consecutive threads walk a tile's column
// (coalesced in column-major C and in the compact partial slots).
template <int BM, int BN>
__global__ void tail_reduce_kernel(i64 M, i64 N, int full, int tail, int tsplits, int gm, int gn, double alpha,
                                   const double* __restrict__ part, double beta, double* __restrict__ C, i64 ldc) {
  constexpr i64 TE = (i64)BM * BN;
  const i64 total = (i64)tail * TE;
  for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
    const int tt = (int)(idx / TE), loc = (int)(idx % TE);
    int tm, tn;
    tile_origin(full + tt, gm, gn, tm, tn);
    const i64 row = (i64)tm * BM + loc % BM, col = (i64)tn * BN + loc / BM;
    if (row >= M || col >= N) continue;
    double s = 0.0;
    for (int z = 0; z < tsplits; ++z) s += part[((i64)z * tail + tt) * TE + loc];
    double* cp = C + row + col * ldc;
    const double v = alpha * s;
    *cp = (beta == 0.0) ? v : v + beta * (*cp);
  }
}

// RUTV_GEMM_SCHED=0 disables the dynamic tile scheduler (static item order)
bool use_sched(const Launch& L) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_GEMM_SCHED");
    v = e ? atoi(e) : 1;
  }
  return v != 0 && L.sched != nullptr;
}

template <class CF, bool TA, bool TB, int VA, int VB, bool CPF>
int launch_t(const Launch& L, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda, const double* B,
             i64 ldb, double beta, double* C, i64 ldc, dim3 grid, i64 kchunk, int full, int tsplits, double* part) {
  RUTV_ONCE_PER_DEVICE(RUTV_CUDA(cudaFuncSetAttribute(
      dgemm_kernel<CF, TA, TB, VA, VB, CPF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM_BYTES)));
  dgemm_kernel<CF, TA, TB, VA, VB, CPF><<<grid, CF::THREADS, CF::SMEM_BYTES, L.stream>>>(M, N, K, alpha, A, lda, B, ldb,
                                                                               beta, C, ldc, kchunk, full, tsplits, part,
                                                                               use_sched(L) ? L.sched : nullptr);
  L.count();
  RUTV_CHECK_LAUNCH("dgemm_kernel");
  return 0;
}

template <class CF, bool TA, bool TB, bool CPF>
int launch_v(const Launch& L, int va, int vb, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
             const double* B, i64 ldb, double beta, double* C, i64 ldc, dim3 grid, i64 kchunk, int full, int tsplits, double* part) {
  if (va == 2 && vb == 2)
    return launch_t<CF, TA, TB, 2, 2, CPF>(L, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  if (va == 2)
    return launch_t<CF, TA, TB, 2, 1, CPF>(L, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  if (vb == 2)
    return launch_t<CF, TA, TB, 1, 2, CPF>(L, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  return launch_t<CF, TA, TB, 1, 1, CPF>(L, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
}

template <class CF, bool TA, bool TB>
int launch_p(const Launch& L, int va, int vb, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
             const double* B, i64 ldb, double beta, double* C, i64 ldc, dim3 grid, i64 kchunk, int full, int tsplits, double* part) {
  // C prefetch instantiation for unsplit read-modify-write epilogues
  // (beta != 0, every item a whole tile)
  if (beta != 0.0 && tsplits == 1)
    return launch_v<CF, TA, TB, true>(L, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  return launch_v<CF, TA, TB, false>(L, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
}

template <class CF>
int launch_cfg(const Launch& L, bool ta, bool tb, int va, int vb, i64 M, i64 N, i64 K, double alpha,
               const double* A, i64 lda, const double* B, i64 ldb, double beta, double* C, i64 ldc, dim3 grid,
               i64 kchunk, int full, int tsplits, double* part) {
  if (!ta && !tb) return launch_p<CF, false, false>(L, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  if (ta && !tb) return launch_p<CF, true, false>(L, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  if (!ta && tb) return launch_p<CF, false, true>(L, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
  return launch_p<CF, true, true>(L, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, full, tsplits, part);
}

// RUTV_GEMM_TAIL=0: no tail-split schedules (unsplit or plain split-K only; A/B)
bool tail_split_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_GEMM_TAIL");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// RUTV_GEMM_PERSIST=0 launches one CTA per tile (tuning comparison only)
bool persistent_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_GEMM_PERSIST");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

inline int vec_of(const double* p, i64 ld) {
  return (((uintptr_t)p & 15) == 0 && (ld % 2) == 0) ? 2 : 1;
}

}  // namespace

namespace {

// The schedule chooser of launch_with as a pure host function (also behind
// randutv_dgemm_plan, so the CPU tests cover it): for `tiles` output tiles of
// bm x bn, `resident` CTA slots and a workspace of ws_elems doubles, the
// number of whole-tile items `full`, the k-ranges per remaining tile
// `tsplits` and their length `kchunk`.  See the comment in launch_with.
void plan_schedule(i64 tiles, i64 K, bool has_ws, i64 ws_elems, i64 resident, int bm, int bn, bool tail_on,
                   i64* full_out, i64* tsplits_out, i64* kchunk_out) {
  const i64 kt = (K + BK - 1) / BK;
  const i64 TE = (i64)bm * bn;
  const double t_kt = 2.0 * bm * bn * BK / (37e12 / (double)resident);  // s per k-tile per item
  i64 full = tiles, tsplits = 1, kchunk = K;
  if (has_ws && K > 0) {
    double best = std::ceil((double)tiles / (double)resident) * (double)kt * t_kt;
    const i64 rem = tiles % resident;
    const i64 cand[3] = {tiles, tail_on ? rem : 0, tail_on ? rem + resident : 0};
    for (int ci = 0; ci < 3; ++ci) {
      const i64 T = cand[ci];
      if (T <= 0 || T > tiles || (ci > 0 && T == tiles)) continue;
      const i64 F = tiles - T;  // a multiple of resident (or 0)
      i64 maxs = ws_elems / (T * TE);
      if (maxs > kt / 4) maxs = kt / 4;  // at least 4 k-tiles (128 of K) per k-range
      if (maxs > 64) maxs = 64;
      for (i64 sp = 2; sp <= maxs; ++sp) {
        const i64 kch = (kt + sp - 1) / sp;
        const double t = (double)(F / resident) * (double)kt * t_kt +
                         std::ceil((double)(T * sp) / (double)resident) * (double)kch * t_kt +
                         (double)(sp + 2) * (double)T * (double)TE * 8.0 / 5e12 + RUTV_SPLIT_FIXED_US * 1e-6;
        const bool ok = ci == 0 || (kt <= 192 && t < best * 0.97);
        if (ok && t < best * (1.0 - 1e-6)) {
          best = t;
          full = F;
          kchunk = kch * BK;
          tsplits = (K + kchunk - 1) / kchunk;
        }
      }
    }
  }
  *full_out = full;
  *tsplits_out = tsplits;
  *kchunk_out = kchunk;
}

template <class CF>
int launch_with(const Launch& L, bool ta, bool tb, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                const double* B, i64 ldb, double beta, double* C, i64 ldc, double* ws, i64 ws_elems) {
  const i64 gm = (M + CF::BM - 1) / CF::BM, gn = (N + CF::BN - 1) / CF::BN;
  const i64 tiles = gm * gn;
  if (tiles > (i64)1 << 30) return -5;
  // resident CTAs.  Whole-tile items all cost the same, so the grid runs in
  // waves of `resident` items and a partial last wave idles the rest of the
  // chip (skinny X W_V at step 48 of c3: 1024 tiles on 444 slots = 2.3 waves).
  // Choose the schedule minimising a time model: waves x k-tiles per item x
  // (one k-tile of one item at peak share) + the reduction of the split
  // tiles (partials written + read at HBM speed, plus a launch).  Candidates:
  // unsplit; the last partial wave (or the last 1.x waves) split into k-ranges
  // that fill the chip (the data-parallel + stream-K hybrid); every tile split
  // (plain split-K).  RUTV_GEMM_TAIL=0 restricts to unsplit / plain split-K.
  // Measured (tools/gemm_shapes.py, profiles/gemm_tail_r02d.txt): the tail
  // split wins on the M = 16384, N = b products with K <= 6144 (c3 step 48
  // X W_V 31.8 -> 34.4 TFLOP/s) but loses ~2 % on long-K ones (step 32
  // A_t^T G: its whole-tile items of 256 k-tiles straggle when residency is
  // uneven), and the c3 step was 0.3 % slower with it unrestricted -- so it is
  // taken only for K <= 6144 and a modelled gain of at least 3 %.
  const i64 resident = (i64)CF::MINB * L.device_sms;
  const i64 TE = (i64)CF::BM * CF::BN;
  i64 full, tsplits, kchunk;
  plan_schedule(tiles, K, ws != nullptr, ws_elems, resident, CF::BM, CF::BN, tail_split_on(), &full, &tsplits, &kchunk);
  if (kchunk <= 0) kchunk = 1;
  const i64 tail = tiles - full;
  const int va = vec_of(A, lda), vb = vec_of(B, ldb);
  const size_t pe = L.pbegin();
  // persistent grid: at most one wave of resident CTAs over all items
  i64 ctas = full + tail * tsplits;
  if (persistent_on() && !L.oneshot && ctas > resident) ctas = resident;
  dim3 grid((unsigned)ctas, 1, 1);
  double* part = tail > 0 ? ws : nullptr;
  RUTV_TRY(launch_cfg<CF>(L, ta, tb, va, vb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, grid, kchunk, (int)full,
                          (int)tsplits, part));
  if (tail > 0) {
    i64 blocks = (tail * TE + 255) / 256;
    if (blocks > (i64)L.device_sms * 8) blocks = (i64)L.device_sms * 8;
    tail_reduce_kernel<CF::BM, CF::BN><<<(unsigned)blocks, 256, 0, L.stream>>>(
        M, N, (int)full, (int)tail, (int)tsplits, (int)gm, (int)gn, alpha, ws, beta, C, ldc);
    L.count();
    RUTV_CHECK_LAUNCH("tail_reduce_kernel");
  }
  // algorithmic: 2MNK flops; compulsory bytes: read A, B (and C if beta != 0), write C
  L.pend(PK_DGEMM, 2.0 * (double)M * (double)N * (double)K,
         8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0.0 ? 2.0 : 1.0)), pe, M, N, K);
  return 0;
}

}  // namespace

// RUTV_GEMM_CFG: "wide" = the 128 x 64 tile for every GEMM, "wide_big" = for
// outputs with both sides >= 1024 only, "wide_skinny" = for skinny long-K
// products only (A/B tuning; default: 64 x 64 -- measured best on the c3 step,
// tools/gpu_session.sh cfg_ab: wide 27.3, wide_big 27.8, default 28.1 TFLOP/s)
static int gemm_cfg_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_GEMM_CFG");
    v = !e ? 0 : (strcmp(e, "wide") == 0 ? 1 : (strcmp(e, "wide_big") == 0 ? 2 : (strcmp(e, "wide_skinny") == 0 ? 3 : 0)));
  }
  return v;
}

int launch_dgemm(const Launch& L, bool ta, bool tb, i64 M, i64 N, i64 K, double alpha, const double* A, i64 lda,
                 const double* B, i64 ldb, double beta, double* C, i64 ldc, double* ws, i64 ws_elems) {
  if (M <= 0 || N <= 0) return 0;
  if (fault_launch()) {
    set_last_error("dgemm_kernel [RUTV_FAULT injected]", cudaErrorLaunchFailure);
    return RANDUTV_ERR_CUDA;
  }
  const int mode = gemm_cfg_mode();
  if (mode == 1 || (mode == 2 && M >= 1024 && N >= 1024) || (mode == 3 && (M <= 512 || N <= 512) && K >= 4096))
    return launch_with<CfgWide>(L, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_elems);
  return launch_with<CfgSmall>(L, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_elems);
}

// randutv_dgemm_plan's body: the default configuration (64 x 64 tiles, 3 CTAs
// per SM) on a device of `sms` SMs; no device needed.
int dgemm_plan(i64 M, i64 N, i64 K, i64 ws_elems, int sms, int tail_on, i64* out) {
  if (M < 0) return -1;
  if (N < 0) return -2;
  if (K < 0) return -3;
  if (ws_elems < 0) return -4;
  if (sms < 1) return -5;
  if (!out) return -7;
  const i64 gm = (M + CfgSmall::BM - 1) / CfgSmall::BM, gn = (N + CfgSmall::BN - 1) / CfgSmall::BN;
  const i64 tiles = gm * gn;
  i64 full = tiles, tsplits = 1, kchunk = K;
  if (tiles > 0)
    plan_schedule(tiles, K, ws_elems > 0, ws_elems, (i64)CfgSmall::MINB * sms, CfgSmall::BM, CfgSmall::BN, tail_on != 0,
                  &full, &tsplits, &kchunk);
  if (kchunk <= 0) kchunk = 1;
  out[0] = tiles;
  out[1] = full;
  out[2] = tsplits;
  out[3] = kchunk;
  out[4] = (i64)CfgSmall::MINB * sms;
  out[5] = (tiles - full) * tsplits * (i64)CfgSmall::BM * CfgSmall::BN;  // workspace doubles the partial tiles take
  return 0;
}

}  // namespace rutv
