// K7 -- S8 of SURVEY.md §8(a): SVD of the b x b diagonal block.
//
// Paper: "Compute the SVD of (U22(:,1:b))* T22 V22(:,1:b) = U_SVD D V_SVD*"
// (Sec. 3.1); FLAME "[A11, U_SVD, V_SVD] := SVD(A11)";
// task Svd_of_block.  The algorithm is reading A10 of DESIGN.md:
// one-sided (Hestenes) Jacobi applied to X = B^T (the ROWS of B are
// orthogonalised, Drmac-Veselic transposition: fast on the row-graded R of a
// randUTV step); at convergence B^T W = Q diag(d), so U_SVD = W, V_SVD = Q.
// A pair (p, q) of columns of X is rotated when
// |x_p.x_q| > tol sqrt(|x_p|^2 |x_q|^2), tol = sqrt(b) 2^-53, with
//   zeta = (beta - alpha)/(2 gamma), t = sign(zeta)/(|zeta| + sqrt(1+zeta^2)),
//   c = 1/sqrt(1+t^2), s = c t,  (x_p, x_q) <- (c x_p - s x_q, s x_p + c x_q),
// columns with |x| <= nu = b 2^-53 ||B||_F are numerically null (never rotated,
// d := 0, completed), stop after a sweep without rotations (cap 30 sweeps ->
// status +block),
// d_j = |x_j|, Q(:,j) = x_j/d_j (zero columns completed by Gram-Schmidt),
// stable descending sort of d.
//
// B200 design.  The oracle visits pairs cyclic-by-rows; here each sweep is the
// b-1 rounds of a round-robin tournament, b/2 disjoint pairs per round, which
// converges to the same d (unique) and to U, V equal up to the signs of
// singular-vector pairs (which no parity metric sees).  X = B^T and
// W = I are split by ROWS over a thread-block cluster of C CTAs (C <= 16,
// chosen so the row slabs fit in shared memory): every column operation is
// row-separable, so each round is
//   1. every CTA: partial (alpha, beta, gamma) of each pair over its rows,
//   2. cluster barrier,
//   3. every CTA: read the C partials of each pair through DSMEM, sum them in
//      rank order (bitwise identical totals, hence identical rotations and
//      identical convergence decisions, in every CTA), rotate its own rows.
// One cluster barrier + one CTA barrier per round; no global memory traffic
// until the factors are written.  Per round: partial Gram entries (thread per
// pair), cluster barrier, the owner CTA of each pair (l mod C) sums the C
// partials in rank order and forms the rotation, cluster barrier, every CTA
// gathers all rotations (one DSMEM load per thread) and rotates its rows.
// Latency-bound: ~2 cluster barriers per round, (b-1) rounds per sweep.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int JT = 256;  // threads per CTA
constexpr int MAX_SWEEPS = 30;

struct JacobiPlan {
  int nc;        // columns incl. phantom (even)
  int C;         // cluster size
  int RP;        // rows per CTA
  int LDS;       // slab column stride (RP + 1: conflict-free when lanes walk columns)
  bool v_smem;   // W slab in shared memory
  size_t smem;   // dynamic smem bytes
};

// shared-memory bytes besides the slabs: part[np][3], rot[np][2], grot[np][2],
// flags (2 x np ints), dsum[nc + 8]
size_t aux_bytes(int nc) {
  const size_t np = nc / 2;
  return np * 3 * 8 + np * 2 * 8 * 2 + np * 4 * 2 + (size_t)(nc + 8) * 8 + 256;
}

JacobiPlan plan_for(i64 w) {
  JacobiPlan p;
  p.nc = (int)(w + (w & 1));
  const size_t limit = 200 * 1024;
  p.C = -1;
  for (int pass = 0; pass < 2; ++pass) {
    for (int C = 1; C <= 16; C *= 2) {
      const int RP = (p.nc + C - 1) / C;
      if (RP > 64) continue;  // apply phase: lanes cover <= 2 rows each
      if ((p.nc / 2 + C - 1) / C > JT) continue;
      const size_t x = (size_t)p.nc * (RP + 1) * 8;
      const size_t need = (pass == 0 ? 2 * x : x) + aux_bytes(p.nc);
      if (need <= limit) {
        p.C = C;
        p.RP = RP;
        p.LDS = RP + 1;
        p.v_smem = pass == 0;
        p.smem = need;
        return p;
      }
    }
  }
  return p;
}

// round-robin tournament: position 0 fixed, positions 1..nc-1 rotate by `round`
__device__ __forceinline__ int rr_col(int pos, int round, int nc) {
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (nc - 1);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// X = B^T (nc x nc, zero padded) split by rows: this CTA holds rows [r0, r0+RP)
// as Xs[col * LDS + lr]; the accumulated rotations W likewise (Ws).
__global__ void __launch_bounds__(JT)
    jacobi_svd_kernel(int w, const double* __restrict__ B, i64 ldb, double* __restrict__ Us, double* __restrict__ d,
                      double* __restrict__ Vs, int* status, int block_id, int nc, int RP, int LDS, int v_smem,
                      double* __restrict__ wglobal, double tol, int* zero_flag) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = JT / 32;
  const int npairs = nc / 2;
  double* Xs = sm;
  double* Ws = v_smem ? Xs + (size_t)nc * LDS : wglobal + (size_t)rank * nc * LDS;
  double* part = v_smem ? Ws + (size_t)nc * LDS : Xs + (size_t)nc * LDS;  // [npairs][3] this CTA's partials
  double* rot = part + npairs * 3;                                        // [npairs][2] owned pairs
  double* grot = rot + npairs * 2;                                        // [npairs][2] gathered
  int* rflag = reinterpret_cast<int*>(grot + npairs * 2);                 // [npairs] owned
  int* gflag = rflag + npairs;                                            // [npairs] gathered
  double* dsum = reinterpret_cast<double*>(gflag + npairs);                // [nc + 8] (2 npairs ints: 8-B aligned)
  __shared__ int sflag[2];
  const int r0 = rank * RP;

  // load X = B^T (zero padded) and W = I for this CTA's rows; partial ||B||_F^2
  double ss = 0.0;
  for (int e = tid; e < nc * RP; e += JT) {
    const int col = e / RP, lr = e % RP, row = r0 + lr;
    const double x = (row < w && col < w) ? B[col + (i64)row * ldb] : 0.0;  // X = B^T
    Xs[col * LDS + lr] = x;
    ss += x * x;
    Ws[col * LDS + lr] = (row == col) ? 1.0 : 0.0;
  }
  ss = warp_sum(ss);
  if (lane == 0) dsum[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < nwarps; ++k) t += dsum[k];
    dsum[nc] = t;  // this CTA's partial, read by every CTA below
  }
  cluster.sync();
  // nu^2 = (w 2^-53 ||B||_F)^2: columns this short are numerically null (not rotated, d := 0)
  double fro2 = 0.0;
  for (int c = 0; c < C; ++c) fro2 += cluster.map_shared_rank(dsum, c)[nc];
  const double nu = (double)w * 0x1p-53 * sqrt(fro2);
  const double nu2 = nu * nu;
  cluster.sync();  // dsum is reused below

  int sweeps = 0;
  bool converged = (nc <= 1);
  const int nown = (npairs - rank + C - 1) / C;  // pairs l = rank + C j owned by this CTA
  while (!converged) {
    if (sweeps >= MAX_SWEEPS) break;
    ++sweeps;
    int rotated = 0;
    for (int round = 0; round < nc - 1; ++round) {
      // 1. partial Gram entries of every pair over this CTA's rows (thread per pair)
      for (int l = tid; l < npairs; l += JT) {
        const int p = rr_col(l, round, nc), q = rr_col(nc - 1 - l, round, nc);
        const double* xp = Xs + p * LDS;
        const double* xq = Xs + q * LDS;
        double a = 0.0, bb = 0.0, g = 0.0;
        for (int lr = 0; lr < RP; ++lr) {
          const double u = xp[lr], v = xq[lr];
          a = fma(u, u, a);
          bb = fma(v, v, bb);
          g = fma(u, v, g);
        }
        part[l * 3 + 0] = a;
        part[l * 3 + 1] = bb;
        part[l * 3 + 2] = g;
      }
      cluster.sync();
      // 2. owners: totals over the cluster in rank order -> rotation of each owned pair
      for (int j = tid; j < nown; j += JT) {
        const int l = rank + C * j;
        double a = 0.0, bb = 0.0, g = 0.0;
        for (int c = 0; c < C; ++c) {
          const double* rp = cluster.map_shared_rank(part + l * 3, c);
          a += rp[0];
          bb += rp[1];
          g += rp[2];
        }
        int f = 0;
        double cs = 1.0, sn = 0.0;
        if (a > nu2 && bb > nu2 && fabs(g) > tol * sqrt(a * bb)) {
          const double zeta = (bb - a) / (2.0 * g);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
          cs = 1.0 / sqrt(1.0 + t * t);
          sn = cs * t;
          f = 1;
        }
        rot[l * 2 + 0] = cs;
        rot[l * 2 + 1] = sn;
        rflag[l] = f;
      }
      cluster.sync();
      // 3. gather every pair's rotation from its owner
      for (int l = tid; l < npairs; l += JT) {
        const int owner = l % C;
        const double* rp = cluster.map_shared_rank(rot + l * 2, owner);
        grot[l * 2 + 0] = rp[0];
        grot[l * 2 + 1] = rp[1];
        gflag[l] = *cluster.map_shared_rank(rflag + l, owner);
      }
      __syncthreads();
      // 4. rotate this CTA's rows of X and W (warp per pair, lanes over rows)
      for (int l = warp; l < npairs; l += nwarps) {
        if (!gflag[l]) continue;
        rotated = 1;
        const int p = rr_col(l, round, nc), q = rr_col(nc - 1 - l, round, nc);
        const double c = grot[l * 2 + 0], s = grot[l * 2 + 1];
        double* xp = Xs + p * LDS;
        double* xq = Xs + q * LDS;
        double* vp = Ws + p * LDS;
        double* vq = Ws + q * LDS;
        for (int lr = lane; lr < RP; lr += 32) {
          const double u = xp[lr], v = xq[lr];
          xp[lr] = c * u - s * v;
          xq[lr] = s * u + c * v;
          const double uu = vp[lr], vv = vq[lr];
          vp[lr] = c * uu - s * vv;
          vq[lr] = s * uu + c * vv;
        }
      }
      __syncthreads();
    }
    converged = __syncthreads_or(rotated) == 0;
  }
  if (!converged && rank == 0 && tid == 0) atomicMin(status, block_id);

  // column norms over the cluster
  for (int col = tid; col < nc; col += JT) {
    const double* xc = Xs + col * LDS;
    double s2 = 0.0;
    for (int lr = 0; lr < RP; ++lr) s2 = fma(xc[lr], xc[lr], s2);
    dsum[col] = s2;
  }
  cluster.sync();
  // every CTA: totals in rank order -> d; ranks for the stable descending sort
  double* dl = part;  // reuse: [nc] totals (part holds 3 npairs >= nc doubles)
  for (int col = tid; col < nc; col += JT) {
    double s2 = 0.0;
    for (int c = 0; c < C; ++c) s2 += cluster.map_shared_rank(dsum, c)[col];
    dl[col] = (s2 <= nu2) ? 0.0 : sqrt(s2);
  }
  if (tid == 0) sflag[0] = 0;
  cluster.sync();  // dsum reads done everywhere; dl visible in this CTA
  for (int col = tid; col < w; col += JT) {
    const double dj = dl[col];
    int rk = 0;
    for (int i = 0; i < nc; ++i) {
      const double di = dl[i];
      rk += (di > dj) || (di == dj && i < col);
    }
    if (rank == 0) d[rk] = dj;
    if (dj == 0.0) sflag[0] = 1;
    const double inv = dj != 0.0 ? 1.0 / dj : 0.0;
    const double* xc = Xs + col * LDS;
    const double* vc = Ws + col * LDS;
    for (int lr = 0; lr < RP; ++lr) {
      const int row = r0 + lr;
      if (row >= w) break;
      Vs[row + (i64)rk * w] = dj != 0.0 ? xc[lr] * inv : 0.0;  // V_SVD = Q = X / d
      Us[row + (i64)rk * w] = vc[lr];                         // U_SVD = W (rotations)
    }
  }
  __syncthreads();
  if (sflag[0] && rank == 0 && tid == 0) atomicExch(zero_flag, 1);
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

}  // namespace

i64 jacobi_scratch_elems(i64 w) {
  const JacobiPlan p = plan_for(w);
  const i64 vg = p.v_smem ? 0 : (i64)p.C * p.nc * p.LDS;
  return vg + w + 64;  // + completion temp + flag
}

int launch_jacobi_svd(const Launch& L, i64 w, const double* B, i64 ldb, double* Us, double* d, double* Vs,
                      int* status, int block_id, double* scratch, i64 scratch_elems) {
  if (w <= 0) return 0;
  const JacobiPlan p = plan_for(w);
  if (p.C <= 0) return -2;
  if (scratch_elems < jacobi_scratch_elems(w)) return -10;
  double* vglobal = p.v_smem ? nullptr : scratch;
  double* ctmp = scratch + (p.v_smem ? 0 : (i64)p.C * p.nc * p.LDS);
  int* zero_flag = reinterpret_cast<int*>(ctmp + w);
  static bool attr_done = false;
  if (!attr_done) {
    RUTV_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    RUTV_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done = true;
  }
  RUTV_CUDA(cudaMemsetAsync(zero_flag, 0, sizeof(int), L.stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.C);
  cfg.blockDim = dim3(JT);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = L.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const double tol = sqrt((double)w) * 0x1p-53;
  const size_t pe = L.pbegin();
  RUTV_CUDA(cudaLaunchKernelEx(&cfg, jacobi_svd_kernel, (int)w, B, ldb, Us, d, Vs, status, block_id, p.nc, p.RP,
                               p.LDS, (int)p.v_smem, vglobal, tol, zero_flag));
  L.count();
  jacobi_complete_kernel<<<1, 256, 0, L.stream>>>((int)w, Vs, d, zero_flag, ctmp);
  L.count();
  RUTV_CHECK_LAUNCH("jacobi_complete_kernel");
  L.pend(PK_JACOBI, 0.0, 8.0 * 4.0 * (double)w * w, pe);
  return 0;
}

}  // namespace rutv
