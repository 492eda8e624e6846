// K1 -- S1 of SURVEY.md §8(a): the Gaussian test matrix G^(i).
//
// Paper: "Draw a random matrix G^(i) in R^{(m-ib) x b}, with i.i.d. entries drawn
// from the standard normal distribution" (Sec. 3.1); FLAME
// ``generate_iid_stdnorm_matrix(m(A) - m(A00), n_b)``.  The
// generator is reading A7 of DESIGN.md: Philox4x32-10 keyed by the 64-bit seed,
// counter (row>>1, col, it, 0); u1 = ((o0:o1) >> 11) 2^-53 + 2^-54,
// u2 = ((o2:o3) >> 11) 2^-53; rho = sqrt(-2 ln u1), theta = 2 pi u2;
// even row -> rho cos(theta), odd row -> rho sin(theta).
//
// One thread per (row pair, column): both Box-Muller outputs of one Philox
// block are used, so each thread writes two adjacent doubles of a column
// (coalesced along the column).  ALU-bound; <0.1% of the factorisation.
#include "common.cuh"

namespace rutv {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__global__ void gaussian_kernel(uint64_t seed, uint32_t it, i64 rows, i64 cols, double* __restrict__ G,
                                i64 ldg) {
  const i64 npairs = (rows + 1) >> 1;
  const i64 total = npairs * cols;
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffull), k1 = (uint32_t)(seed >> 32);
  for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
    const i64 p = idx % npairs;
    const i64 c = idx / npairs;
    uint32_t ctr[4] = {(uint32_t)p, (uint32_t)c, it, 0u};
    philox4x32_10(ctr, k0, k1);
    const uint64_t w1 = ((uint64_t)ctr[0] << 32) | ctr[1];
    const uint64_t w2 = ((uint64_t)ctr[2] << 32) | ctr[3];
    const double u1 = (double)(w1 >> 11) * 0x1p-53 + 0x1p-54;
    const double u2 = (double)(w2 >> 11) * 0x1p-53;
    const double rho = sqrt(-2.0 * log(u1));
    const double theta = 6.283185307179586 * u2;
    double s, co;
    sincos(theta, &s, &co);
    const i64 r0 = 2 * p;
    double* col = G + c * ldg;
    col[r0] = rho * co;
    if (r0 + 1 < rows) col[r0 + 1] = rho * s;
  }
}

int launch_gaussian(const Launch& L, uint64_t seed, i64 it, i64 rows, i64 cols, double* G, i64 ldg) {
  if (rows <= 0 || cols <= 0) return 0;
  const i64 total = ((rows + 1) >> 1) * cols;
  const int threads = 256;
  i64 blocks = (total + threads - 1) / threads;
  if (blocks > (i64)L.device_sms * 16) blocks = (i64)L.device_sms * 16;
  const size_t pe = L.pbegin();
  gaussian_kernel<<<(unsigned)blocks, threads, 0, L.stream>>>(seed, (uint32_t)it, rows, cols, G, ldg);
  L.count();
  L.pend(PK_GAUSSIAN, 0.0, 8.0 * (double)rows * cols, pe);
  RUTV_CHECK_LAUNCH("gaussian_kernel");
  return 0;
}

}  // namespace rutv
