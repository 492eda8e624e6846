#include <cstdlib>
// K7 -- S8 of SURVEY.md §8(a): SVD of the b x b diagonal block.
//
// Paper: "Compute the SVD of (U22(:,1:b))* T22 V22(:,1:b) = U_SVD D V_SVD*"
// (Sec. 3.1); FLAME "[A11, U_SVD, V_SVD] := SVD(A11)";
// task Svd_of_block.  The algorithm is reading A10/A23/A24 of
// one-sided (Hestenes) Jacobi applied to X = B^T (the ROWS of B are
// orthogonalised); at convergence B^T W = Q diag(d), so U_SVD = W, V_SVD = Q.
// A pair (p, q) of columns of X is rotated when both columns are longer than
// nu = b 2^-53 ||B||_F and |x_p.x_q| > tol sqrt(|x_p|^2 |x_q|^2),
// tol = sqrt(b) 2^-53, with
//   zeta = (beta - alpha)/(2 gamma), t = sign(zeta)/(|zeta| + sqrt(1+zeta^2)),
//   c = 1/sqrt(1+t^2), s = c t,  (x_p, x_q) <- (c x_p - s x_q, s x_p + c x_q);
// stop after a sweep without rotations (cap 30 sweeps -> status +block);
// d_j = |x_j| (0 if |x_j| <= nu), Q(:,j) = x_j/d_j (zero columns completed by
// Gram-Schmidt); stable descending sort of d.
//
// B200 design: BLOCK one-sided Jacobi (reading A25: a different, equally valid
// cyclic pair order than the oracle's; same d, U/V up to singular-vector signs).
// The nc columns of X (b padded to a multiple of 2 nb with zero columns) form
// nblk = nc/nb column blocks; P = nblk/2 CTAs of a cooperative grid each take a
// pair of blocks per block round (round-robin tournament over blocks, nblk-1
// block rounds per sweep), stage their 2 nb columns of X and of W in shared
// memory, and perform every cross pair (p in I, q in J) as nb inner rounds of
// nb disjoint rotations (intra-block pairs in the first block round of a
// sweep) -- warp per pair, lanes over rows, so the per-rotation barrier is a
// CTA barrier, not a grid/cluster one.  One grid barrier per block round.
// Every pair is visited once per sweep; each dot product is one warp's fixed
// lane-strided sum + xor butterfly (bitwise identical on every lane and run).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

#ifndef RUTV_JT
#define RUTV_JT 512
#endif
constexpr int JT = RUTV_JT;  // threads per CTA
constexpr int MAX_SWEEPS = 30;

struct JacobiPlan {
  int nb;      // columns per block
  int nc;      // padded column count (multiple of 2 nb)
  int P;       // CTAs = nblk / 2
  size_t smem; // dynamic shared memory
};

JacobiPlan plan_for(i64 w) {
  JacobiPlan p;
  p.nb = 8;  // 16 for w <= 256 was measured 15-20 % slower (more CTAs per block round win)
  {
    static int env_nb = -1;  // RUTV_JNB: block width override (tuning only)
    if (env_nb < 0) {
      const char* e = getenv("RUTV_JNB");
      env_nb = e ? atoi(e) : 0;
    }
    if (env_nb > 0 && 2 * (i64)env_nb * ((w < 1 ? 1 : w) + w + 2 * env_nb) * 8 <= 200 * 1024) p.nb = env_nb;
  }
  const i64 ww = w < 1 ? 1 : w;
  p.nc = (int)((ww + 2 * p.nb - 1) / (2 * p.nb) * (2 * p.nb));
  p.P = p.nc / p.nb / 2;
  p.smem = (size_t)2 * p.nb * ((size_t)ww + p.nc) * sizeof(double);
  return p;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// RUTV_JACOBI_CLUSTER=0 forces the L2-staged cooperative kernel for w <= 256 (A/B only)
bool jacobi_cluster_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_JACOBI_CLUSTER");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// round-robin tournament over `n` (even) slots: slot 0 fixed, others rotate
__device__ __forceinline__ int rr(int pos, int round, int n) {
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (n - 1);
}

// One warp: test and (maybe) rotate the column pair (xp, xq) of X (w rows) and
// (wp, wq) of W (nc rows).  Returns 1 if rotated.
__device__ __forceinline__ int jacobi_pair(double* xp, double* xq, double* wp, double* wq, int w, int nc,
                                           double tol, double nu2, int lane) {
  double a = 0.0, bb = 0.0, g = 0.0;
  for (int r = lane; r < w; r += 32) {
    const double u = xp[r], v = xq[r];
    a = fma(u, u, a);
    bb = fma(v, v, bb);
    g = fma(u, v, g);
  }
  a = warp_sum(a);
  bb = warp_sum(bb);
  g = warp_sum(g);
  // |g| > tol sqrt(a bb) without the square root (FP64 sqrt / division are
  // the long-latency steps of a rotation; a, bb > nu2 keep the product in range)
  if (!(a > nu2 && bb > nu2 && g * g > (tol * tol) * (a * bb))) return 0;
  // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (bb - a) / (2 g),
  // written as 2 g sign(bb - a) / (|bb - a| + sqrt((bb - a)^2 + 4 g^2)): one
  // square root and one division; c = 1 / sqrt(1 + t^2) by rsqrt
  const double dba = bb - a;
  const double t = copysign(1.0, dba) * (2.0 * g) / (fabs(dba) + sqrt(fma(dba, dba, 4.0 * g * g)));
  const double c = rsqrt(fma(t, t, 1.0));
  const double s = c * t;
  for (int r = lane; r < w; r += 32) {
    const double u = xp[r], v = xq[r];
    xp[r] = c * u - s * v;
    xq[r] = s * u + c * v;
  }
  for (int r = lane; r < nc; r += 32) {
    const double u = wp[r], v = wq[r];
    wp[r] = c * u - s * v;
    wq[r] = s * u + c * v;
  }
  return 1;
}

// The cluster kernel's rotation on register-resident columns.  Shared memory
// bandwidth (128 B/clk/SM) bounded the pair above: eight warps each reading and
// writing two X and two W columns per inner round (~128 KB, ~1000 cycles of a
// ~2500-cycle round).  Here (u, v) are the X columns in registers (K per lane;
// the caller keeps the slot-0 column of its warp resident across the cross
// rounds), and the W columns are not touched: the rotation is accumulated
// into the CTA's 16 x 16 factor Jm (column-major, J <- J R on columns jp, jq;
// 16 lanes) and W <- W J is applied once per block round.
template <int K>
__device__ __forceinline__ int jacobi_rot_reg(double (&u)[K], double (&v)[K], double tol, double nu2, int lane,
                                              double* Jm, int jp, int jq) {
  double a = 0.0, bb = 0.0, g = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    a = fma(u[k], u[k], a);
    bb = fma(v[k], v[k], bb);
    g = fma(u[k], v[k], g);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ta = __shfl_xor_sync(0xffffffffu, a, o);
    const double tb = __shfl_xor_sync(0xffffffffu, bb, o);
    const double tg = __shfl_xor_sync(0xffffffffu, g, o);
    a += ta;
    bb += tb;
    g += tg;
  }
  if (!(a > nu2 && bb > nu2 && g * g > (tol * tol) * (a * bb))) return 0;
  const double dba = bb - a;
  const double den = fabs(dba) + sqrt(fma(dba, dba, 4.0 * g * g));
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(den));
  y = fma(y, fma(-den, y, 1.0), y);
  y = fma(y, fma(-den, y, 1.0), y);
  const double t = copysign(1.0, dba) * (2.0 * g) * y;
  const double c = rsqrt(fma(t, t, 1.0));
  const double s = c * t;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double x = u[k], z = v[k];
    u[k] = c * x - s * z;
    v[k] = s * x + c * z;
  }
  if (lane < 16) {
    const double x = Jm[jp * 16 + lane], z = Jm[jq * 16 + lane];
    Jm[jp * 16 + lane] = c * x - s * z;
    Jm[jq * 16 + lane] = s * x + c * z;
  }
  return 1;
}

template <int K>
__device__ __forceinline__ void col_load(double (&u)[K], const double* x, int w, int lane) {
#pragma unroll
  for (int k = 0; k < K; ++k) u[k] = lane + 32 * k < w ? x[lane + 32 * k] : 0.0;
}
template <int K>
__device__ __forceinline__ void col_store(const double (&u)[K], double* x, int w, int lane) {
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (lane + 32 * k < w) x[lane + 32 * k] = u[k];
}

// Xg: w x nc (X = B^T, zero padded columns), Wg: nc x nc, both column-major in
// global memory (L2 resident).  red: >= 2 P + nc doubles; flags: MAX_SWEEPS+1 ints (zeroed).
__global__ void __launch_bounds__(JT)
    jacobi_block_kernel(int w, const double* __restrict__ B, i64 ldb, double* __restrict__ Us, double* __restrict__ d,
                        double* __restrict__ Vs, int* status, int block_id, int nb, int nc, double* __restrict__ Xg,
                        double* __restrict__ Wg, double* __restrict__ red, int* __restrict__ flags, double tol,
                        int* zero_flag, int max_sweeps) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  __shared__ double wred[JT / 32];
  __shared__ int srot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = JT / 32;
  const int cta = blockIdx.x, P = gridDim.x;
  const int nblk = nc / nb;
  double* Xs = sm;                       // 2 nb columns x w
  double* Ws = sm + (size_t)2 * nb * w;  // 2 nb columns x nc

  // ---- X = B^T, W = I; this CTA initialises columns [cta*2nb, (cta+1)*2nb)
  double ss = 0.0;
  for (int cl = 0; cl < 2 * nb; ++cl) {
    const int col = cta * 2 * nb + cl;
    for (int r = tid; r < w; r += JT) {
      const double x = col < w ? B[col + (i64)r * ldb] : 0.0;
      Xg[r + (i64)col * w] = x;
      ss = fma(x, x, ss);
    }
    for (int r = tid; r < nc; r += JT) Wg[r + (i64)col * nc] = (r == col) ? 1.0 : 0.0;
  }
  ss = warp_sum(ss);
  if (lane == 0) wred[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < nwarps; ++k) t += wred[k];
    red[cta] = t;
  }
  grid.sync();
  double fro2 = 0.0;
  for (int c = 0; c < P; ++c) fro2 += red[c];  // same order in every CTA
  const double nu = (double)w * 0x1p-53 * sqrt(fro2);
  const double nu2 = nu * nu;

  int sweeps = 0;
  bool converged = (w <= 1);
  while (!converged) {
    if (sweeps >= max_sweeps) break;
    int rotated = 0;
    for (int r = 0; r < nblk - 1; ++r) {
      const int I = rr(cta, r, nblk), J = rr(nblk - 1 - cta, r, nblk);
      // stage blocks I and J of X and W: cp.async, every element in flight at once
      {
        const double* xI = Xg + (i64)I * nb * w;
        const double* xJ = Xg + (i64)J * nb * w;
        const double* wI = Wg + (i64)I * nb * nc;
        const double* wJ = Wg + (i64)J * nb * nc;
        const int nx = nb * w, nw = nb * nc;
        for (int e = tid; e < nx; e += JT) {
          cp_async8(Xs + e, xI + e);
          cp_async8(Xs + nx + e, xJ + e);
        }
        for (int e = tid; e < nw; e += JT) {
          cp_async8(Ws + e, wI + e);
          cp_async8(Ws + nw + e, wJ + e);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      }
      __syncthreads();
      if (r == 0) {
        // intra-block pairs of both blocks: nb-1 inner rounds, nb/2 pairs per block each
        for (int t = 0; t < nb - 1; ++t) {
          for (int pi = warp; pi < nb; pi += nwarps) {
            const int blk = pi / (nb / 2), k = pi % (nb / 2);
            const int p = blk * nb + rr(k, t, nb), q = blk * nb + rr(nb - 1 - k, t, nb);
            rotated |= jacobi_pair(Xs + (size_t)p * w, Xs + (size_t)q * w, Ws + (size_t)p * nc, Ws + (size_t)q * nc,
                                   w, nc, tol, nu2, lane);
          }
          __syncthreads();
        }
      }
      // cross pairs (a in I, (a + t) mod nb in J): nb inner rounds of nb disjoint pairs
      for (int t = 0; t < nb; ++t) {
        for (int a = warp; a < nb; a += nwarps) {
          const int p = a, q = nb + (a + t) % nb;
          rotated |= jacobi_pair(Xs + (size_t)p * w, Xs + (size_t)q * w, Ws + (size_t)p * nc, Ws + (size_t)q * nc, w,
                                 nc, tol, nu2, lane);
        }
        __syncthreads();
      }
      {
        double* xI = Xg + (i64)I * nb * w;
        double* xJ = Xg + (i64)J * nb * w;
        double* wI = Wg + (i64)I * nb * nc;
        double* wJ = Wg + (i64)J * nb * nc;
        const int nx = nb * w, nw = nb * nc;
        for (int e = tid; e < nx; e += JT) {
          xI[e] = Xs[e];
          xJ[e] = Xs[nx + e];
        }
        for (int e = tid; e < nw; e += JT) {
          wI[e] = Ws[e];
          wJ[e] = Ws[nw + e];
        }
      }
      grid.sync();
    }
    if (tid == 0) srot = 0;
    __syncthreads();
    if (rotated) atomicOr(&srot, 1);
    __syncthreads();
    if (tid == 0 && srot) atomicOr(&flags[sweeps], 1);
    grid.sync();
    converged = (*(volatile int*)&flags[sweeps]) == 0;
    ++sweeps;
  }
  if (!converged && cta == 0 && tid == 0) atomicMin(status, block_id);

  // ---- column norms (thread per column, sequential over rows), d, stable descending sort
  double* dn = red + 2 * P;  // [nc]
  for (int col = cta * nwarps + warp; col < nc; col += P * nwarps) {  // warp per column
    const double* xc = Xg + (i64)col * w;
    double s2 = 0.0;
    for (int e = lane; e < w; e += 32) s2 = fma(xc[e], xc[e], s2);
    s2 = warp_sum(s2);
    if (lane == 0) dn[col] = (s2 <= nu2) ? 0.0 : sqrt(s2);
  }
  grid.sync();
  int anyzero = 0;
  for (int col = cta; col < w; col += P) {  // CTA per column
    const double dj = dn[col];
    int rk = 0;
    for (int i = tid; i < nc; i += JT) {
      const double di = dn[i];
      rk += (di > dj) || (di == dj && i < col);
    }
    rk = __reduce_add_sync(0xffffffffu, rk);
    if (lane == 0) wred[warp] = (double)rk;
    __syncthreads();
    int rank = 0;
    for (int k = 0; k < nwarps; ++k) rank += (int)wred[k];
    __syncthreads();
    if (tid == 0) d[rank] = dj;
    anyzero |= (dj == 0.0);
    const double inv = dj != 0.0 ? 1.0 / dj : 0.0;
    for (int e = tid; e < w; e += JT) {
      Vs[e + (i64)rank * w] = dj != 0.0 ? Xg[e + (i64)col * w] * inv : 0.0;  // V_SVD = Q = X / d
      Us[e + (i64)rank * w] = Wg[e + (i64)col * nc];                         // U_SVD = W
    }
  }
  if (anyzero && tid == 0) atomicExch(zero_flag, 1);
}

// Completion of the Q (= V_SVD) columns with d_j == 0 (sorted last): Gram-Schmidt of e_1, e_2, ...
// against the columns present (twice), as the oracle.  Runs only if flagged.
__global__ void jacobi_complete_kernel(int w, double* __restrict__ Us, const double* __restrict__ d,
                                       int* zero_flag, double* __restrict__ tmp) {
  if (*zero_flag == 0) return;
  __shared__ double red[32];
  __shared__ int accept;
  const int tid = threadIdx.x;
  int e = 0;
  int first_zero = w;
  for (int j = 0; j < w; ++j)
    if (d[j] == 0.0) { first_zero = j; break; }
  for (int j = first_zero; j < w; ++j) {
    while (true) {
      if (e >= w) return;
      for (int r = tid; r < w; r += blockDim.x) tmp[r] = (r == e) ? 1.0 : 0.0;
      __syncthreads();
      ++e;
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i < j; ++i) {
          double s = 0.0;
          for (int r = tid; r < w; r += blockDim.x) s += Us[r + (i64)i * w] * tmp[r];
          s = warp_sum(s);
          if ((tid & 31) == 0) red[tid >> 5] = s;
          __syncthreads();
          if (tid == 0) {
            double t = 0.0;
            for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += red[k];
            red[0] = t;
          }
          __syncthreads();
          const double proj = red[0];
          __syncthreads();
          for (int r = tid; r < w; r += blockDim.x) tmp[r] -= proj * Us[r + (i64)i * w];
          __syncthreads();
        }
      }
      double s = 0.0;
      for (int r = tid; r < w; r += blockDim.x) s += tmp[r] * tmp[r];
      s = warp_sum(s);
      if ((tid & 31) == 0) red[tid >> 5] = s;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += red[k];
        red[0] = sqrt(t);
        accept = red[0] > 0.5;
      }
      __syncthreads();
      const double nx = red[0];
      if (accept) {
        for (int r = tid; r < w; r += blockDim.x) Us[r + (i64)j * w] = tmp[r] / nx;
        __syncthreads();
        break;
      }
      __syncthreads();
    }
  }
  if (tid == 0) *zero_flag = 0;
}

// ---------------------------------------------------------------------------
// w <= 256: the same block Jacobi with the data RESIDENT in one thread-block
// cluster (P = nc / 16 <= 16 CTAs, non-portable size).  CTA c keeps the X and
// W columns of the two blocks at tournament positions c and 2P-1-c in its own
// shared memory for the whole SVD; after every block round the blocks move one
// position (slot 0 fixed, the others rotate -- the round-robin schedule of
// rr()), each CTA copying its two incoming blocks from the neighbours'
// shared memory over DSMEM into its second buffer.  One cluster barrier per
// block round, no L2 round trips, no grid barrier.  Same pair order and
// arithmetic as jacobi_block_kernel.
constexpr int JCT = 256;  // threads per cluster CTA: one warp per pair (nb = 8)

__global__ void __launch_bounds__(JCT, 1)
    jacobi_cluster_kernel(int w, const double* __restrict__ B, i64 ldb, double* __restrict__ Us,
                          double* __restrict__ d, double* __restrict__ Vs, int* status, int block_id, int nb, int nc,
                          double tol, int* zero_flag, int max_sweeps) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  __shared__ double wred[JCT / 32];
  __shared__ double part;       // this CTA's sum of squares of B
  __shared__ int rotf[2];       // rotations in the sweep, by sweep parity
  __shared__ double dn[2 * 8];  // this CTA's column norms (2 nb <= 16)
  __shared__ double dall[256];  // every column norm (global column order)
  __shared__ int srot;
  __shared__ double Jm[256];    // the block round's W rotation (16 x 16, column-major)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = JCT / 32;
  const int cta = (int)cl.block_rank(), P = (int)cl.num_blocks();
  const int nblk = 2 * P;
  const int sx = nb * w, sw = nb * nc, slot = sx + sw;  // one block: X (nb x w) then W (nb x nc)
  double* buf[2] = {sm, sm + 2 * slot};

  // ---- X = B^T, W = I for the blocks at positions cta (slot 0) and nblk-1-cta (slot 1)
  double ss = 0.0;
  for (int sl = 0; sl < 2; ++sl) {
    const int blk = sl == 0 ? cta : nblk - 1 - cta;
    double* X = buf[0] + sl * slot;
    double* W = X + sx;
    for (int e = tid; e < sx; e += JCT) {
      const int cl_ = e / w, r = e % w, col = blk * nb + cl_;
      const double x = col < w ? B[col + (i64)r * ldb] : 0.0;
      X[e] = x;
      ss = fma(x, x, ss);
    }
    for (int e = tid; e < sw; e += JCT) {
      const int cl_ = e / nc, r = e % nc, col = blk * nb + cl_;
      W[e] = (r == col) ? 1.0 : 0.0;
    }
  }
  ss = warp_sum(ss);
  if (lane == 0) wred[warp] = ss;
  if (tid < 2) rotf[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < nwarps; ++k) t += wred[k];
    part = t;
  }
  cl.sync();
  double fro2 = 0.0;
  for (int c = 0; c < P; ++c) fro2 += *cl.map_shared_rank(&part, c);  // same order in every CTA
  const double nu = (double)w * 0x1p-53 * sqrt(fro2);
  const double nu2 = nu * nu;

  // sources of the two incoming blocks after a round (positions move p -> p-1,
  // 1 -> nblk-1, 0 fixed): slot 0 <- position cta+1, slot 1 <- position nblk-cta
  int src0_rank = cta, src0_slot = 0, src1_rank = 0, src1_slot = 0;
  if (cta > 0) {
    if (cta + 1 <= P - 1) src0_rank = cta + 1, src0_slot = 0;
    else src0_rank = P - 1, src0_slot = 1;  // position P = nblk-1-(P-1)
  }
  if (cta == 0) src1_rank = P > 1 ? 1 : 0, src1_slot = 0;  // position nblk-1 <- position 1
  else src1_rank = cta - 1, src1_slot = 1;

  int cur = 0, sweeps = 0;
  bool converged = (w <= 1);
  while (!converged) {
    if (sweeps >= max_sweeps) break;
    int rotated = 0;
    for (int r = 0; r < nblk - 1; ++r) {
      double* Xs = buf[cur];          // slot 0 X at Xs, slot 1 X at Xs + slot
      double* X0 = Xs;
      double* X1 = Xs + slot;
      double* W0 = X0 + sx;
      double* W1 = X1 + sx;
      // J := I (the block round's accumulated W rotation, 16 x 16)
      for (int e = tid; e < 256; e += JCT) Jm[e] = (e % 17 == 0) ? 1.0 : 0.0;
      __syncthreads();
      if (r == 0) {
        // intra-block pairs of both blocks: nb-1 inner rounds, nb/2 pairs per block (warp = pair)
        for (int t = 0; t < nb - 1; ++t) {
          const int blk = warp / (nb / 2), k = warp % (nb / 2);
          const int p = rr(k, t, nb), q = rr(nb - 1 - k, t, nb);
          double* Xb = blk == 0 ? X0 : X1;
          double u[8], v[8];
          col_load<8>(u, Xb + (size_t)p * w, w, lane);
          col_load<8>(v, Xb + (size_t)q * w, w, lane);
          if (jacobi_rot_reg<8>(u, v, tol, nu2, lane, Jm, blk * nb + p, blk * nb + q)) {
            rotated = 1;
            col_store<8>(u, Xb + (size_t)p * w, w, lane);
            col_store<8>(v, Xb + (size_t)q * w, w, lane);
          }
          __syncthreads();
        }
      }
      // cross pairs (a in slot 0, (a + t) mod nb in slot 1): nb inner rounds of
      // nb disjoint pairs; warp a keeps slot-0 column a in registers throughout
      {
        const int a = warp;
        double u[8];
        col_load<8>(u, X0 + (size_t)a * w, w, lane);
        for (int t = 0; t < nb; ++t) {
          const int q = (a + t) % nb;
          double v[8];
          col_load<8>(v, X1 + (size_t)q * w, w, lane);
          if (jacobi_rot_reg<8>(u, v, tol, nu2, lane, Jm, a, nb + q)) {
            rotated = 1;
            col_store<8>(v, X1 + (size_t)q * w, w, lane);
          }
          __syncthreads();
        }
        col_store<8>(u, X0 + (size_t)a * w, w, lane);
      }
      // W <- W J over the 16 columns [W0 | W1]: DMMA m8n8k4, warp per 8-row
      // block (both 8-column halves), fragments straight from shared memory;
      // a warp reads all 16 columns of its rows before the mma writes them
      for (int rb8 = warp; rb8 * 8 < nc; rb8 += nwarps) {
        const int row = rb8 * 8 + (lane >> 2), t4 = lane & 3;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int k = kk * 4 + t4;  // column of [W0 | W1]
          const double av = k < nb ? W0[(size_t)k * nc + row] : W1[(size_t)(k - nb) * nc + row];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            const double bv = Jm[(ni * 8 + (lane >> 2)) * 16 + k];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[ni][0]), "+d"(acc[ni][1])
                         : "d"(av), "d"(bv));
          }
        }
        // lane (g, t4) holds rows rb8*8 + g, columns ni*8 + 2 t4 + {0, 1}: W0 for ni = 0, W1 for ni = 1
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          double* Wd = ni == 0 ? W0 : W1;
          Wd[(size_t)(2 * t4) * nc + row] = acc[ni][0];
          Wd[(size_t)(2 * t4 + 1) * nc + row] = acc[ni][1];
        }
      }
      __syncthreads();
      if (nblk > 2) {
        // rotate the tournament: fetch the two incoming blocks into the other buffer
        cl.sync();
        double* dst = buf[cur ^ 1];
        const double* s0 = cl.map_shared_rank(buf[cur] + src0_slot * slot, src0_rank);
        const double* s1 = cl.map_shared_rank(buf[cur] + src1_slot * slot, src1_rank);
        // 16-byte DSMEM loads, four per thread in flight before the stores
        const double2* a2 = reinterpret_cast<const double2*>(s0);
        const double2* b2 = reinterpret_cast<const double2*>(s1);
        double2* d2 = reinterpret_cast<double2*>(dst);
        const int h2 = slot / 2;
        for (int e0 = tid; e0 < h2; e0 += 2 * JCT) {
          const int e1 = e0 + JCT;
          const double2 x0 = a2[e0], y0 = b2[e0];
          double2 x1 = make_double2(0.0, 0.0), y1 = x1;
          if (e1 < h2) {
            x1 = a2[e1];
            y1 = b2[e1];
          }
          d2[e0] = x0;
          d2[h2 + e0] = y0;
          if (e1 < h2) {
            d2[e1] = x1;
            d2[h2 + e1] = y1;
          }
        }
        __syncthreads();
        cur ^= 1;
      }
    }
    // sweep verdict: any rotation in any CTA
    if (tid == 0) srot = 0;
    __syncthreads();
    if (rotated) atomicOr(&srot, 1);
    __syncthreads();
    if (tid == 0) rotf[sweeps & 1] = srot;
    cl.sync();
    int any = 0;
    for (int c = 0; c < P; ++c) any |= *cl.map_shared_rank(&rotf[sweeps & 1], c);
    converged = any == 0;
    ++sweeps;
  }
  if (!converged && cta == 0 && tid == 0) atomicMin(status, block_id);
#ifdef RUTV_JACOBI_PROF
  if (cta == 0 && tid == 0) printf("jacobi_cluster w=%d P=%d sweeps=%d\n", w, P, sweeps);
#endif

  // ---- column norms, global ranks (stable descending), outputs
  double* Xc = buf[cur];
  for (int cl_ = warp; cl_ < 2 * nb; cl_ += nwarps) {
    const double* xc = Xc + (cl_ / nb) * slot + (size_t)(cl_ % nb) * w;
    double s2 = 0.0;
    for (int e = lane; e < w; e += 32) s2 = fma(xc[e], xc[e], s2);
    s2 = warp_sum(s2);
    if (lane == 0) dn[cl_] = (s2 <= nu2) ? 0.0 : sqrt(s2);
  }
  cl.sync();
  for (int col = tid; col < nc; col += JCT) {
    const int blk = col / nb, i = col % nb;
    const int owner = blk < P ? blk : nblk - 1 - blk, sl = blk < P ? 0 : 1;
    dall[col] = *cl.map_shared_rank(&dn[sl * nb + i], owner);
  }
  __syncthreads();
  int anyzero = 0;
  for (int cl_ = 0; cl_ < 2 * nb; ++cl_) {
    const int blk = cl_ < nb ? cta : nblk - 1 - cta;
    const int col = blk * nb + cl_ % nb;
    if (col >= w) continue;
    const double dj = dall[col];
    int rk = 0;
    for (int i = tid; i < nc; i += JCT) {
      const double di = dall[i];
      rk += (di > dj) || (di == dj && i < col);
    }
    rk = __reduce_add_sync(0xffffffffu, rk);
    if (lane == 0) wred[warp] = (double)rk;
    __syncthreads();
    int rank = 0;
    for (int k = 0; k < nwarps; ++k) rank += (int)wred[k];
    __syncthreads();
    if (tid == 0) d[rank] = dj;
    anyzero |= (dj == 0.0);
    const double inv = dj != 0.0 ? 1.0 / dj : 0.0;
    const double* xc = Xc + (cl_ / nb) * slot + (size_t)(cl_ % nb) * w;
    const double* wc = Xc + (cl_ / nb) * slot + sx + (size_t)(cl_ % nb) * nc;
    for (int e = tid; e < w; e += JCT) {
      Vs[e + (i64)rank * w] = dj != 0.0 ? xc[e] * inv : 0.0;  // V_SVD = Q = X / d
      Us[e + (i64)rank * w] = wc[e];                         // U_SVD = W
    }
  }
  if (anyzero && tid == 0) atomicExch(zero_flag, 1);
  cl.sync();  // no CTA exits while its shared memory may still be read
}

}  // namespace

i64 jacobi_scratch_elems(i64 w) {
  const JacobiPlan p = plan_for(w);
  const i64 ww = w < 1 ? 1 : w;
  // Xg (w x nc) + Wg (nc x nc) + red (2P + nc) + completion temp (w) + flags/zero flag
  return ww * p.nc + (i64)p.nc * p.nc + 2 * p.P + p.nc + ww + 64;
}

int launch_jacobi_svd(const Launch& L, i64 w, const double* B, i64 ldb, double* Us, double* d, double* Vs,
                      int* status, int block_id, double* scratch, i64 scratch_elems) {
  if (w <= 0) return 0;
  const JacobiPlan p = plan_for(w);
  if (scratch_elems < jacobi_scratch_elems(w)) return -10;
  double* Xg = scratch;
  double* Wg = Xg + w * p.nc;
  double* red = Wg + (i64)p.nc * p.nc;
  double* ctmp = red + 2 * p.P + p.nc;
  int* iflags = reinterpret_cast<int*>(ctmp + w);  // [0] zero flag, [1..] sweep flags
  int* zero_flag = iflags;
  int* flags = iflags + 1;
  RUTV_ONCE_PER_DEVICE(
      RUTV_CUDA(cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)));
  RUTV_CUDA(cudaMemsetAsync(iflags, 0, sizeof(int) * (MAX_SWEEPS + 2), L.stream));
  const size_t pe = L.pbegin();
  const int msw0 = L.jacobi_max_sweeps < 1 ? 1 : (L.jacobi_max_sweeps > MAX_SWEEPS ? MAX_SWEEPS : L.jacobi_max_sweeps);
  // the cluster variant (16-byte DSMEM exchange) measured at or below the
  // L2-staged kernel for every w <= 256 (64: 0.56 vs 0.65 ms, 128: 1.48 vs
  // 1.63, 256: 4.71 vs 4.75; tools/gpu_session.sh leaf_ab)
  if (w <= 256 && jacobi_cluster_on()) {
    // data-resident cluster variant: nb = 8, P = nc / 16 CTAs (<= 16)
    const int nb = 8, nc = (int)((w + 15) / 16 * 16), P = nc / 16;
    const size_t smem = (size_t)4 * nb * ((size_t)w + nc) * sizeof(double);
    RUTV_ONCE_PER_DEVICE({
      RUTV_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      RUTV_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     4 * 8 * 512 * 8));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(JCT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = L.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RUTV_CUDA(cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel, (int)w, B, (i64)ldb, Us, d, Vs, status, block_id, nb, nc,
                                 sqrt((double)w) * 0x1p-53, zero_flag, msw0));
    L.count();
    jacobi_complete_kernel<<<1, 256, 0, L.stream>>>((int)w, Vs, d, zero_flag, ctmp);
    L.count();
    RUTV_CHECK_LAUNCH("jacobi_complete_kernel");
    L.pend(PK_JACOBI, 0.0, 8.0 * 4.0 * (double)w * w, pe);
    return 0;
  }
  int wi = (int)w, bid = block_id, nbv = p.nb, ncv = p.nc;
  i64 ldbv = ldb;
  double tol = sqrt((double)w) * 0x1p-53;
  const double* Bv = B;
  int msw = L.jacobi_max_sweeps < 1 ? 1 : (L.jacobi_max_sweeps > MAX_SWEEPS ? MAX_SWEEPS : L.jacobi_max_sweeps);
  void* args[] = {&wi, &Bv, &ldbv, &Us, &d, &Vs, &status, &bid, &nbv, &ncv, &Xg, &Wg, &red, &flags, &tol, &zero_flag,
                  &msw};
  RUTV_CUDA(cudaLaunchCooperativeKernel((void*)jacobi_block_kernel, dim3(p.P), dim3(JT), args, p.smem, L.stream));
  L.count();
  jacobi_complete_kernel<<<1, 256, 0, L.stream>>>((int)w, Vs, d, zero_flag, ctmp);
  L.count();
  RUTV_CHECK_LAUNCH("jacobi_complete_kernel");
  L.pend(PK_JACOBI, 0.0, 8.0 * 4.0 * (double)w * w, pe);
  return 0;
}

}  // namespace rutv
