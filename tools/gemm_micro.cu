// DMMA main-loop microbenchmark (tuning tool, not part of the library): the
// shared-memory fragment loads + mma.sync.m8n8k4.f64 pattern of dgemm_kernel in
// isolation (operands resident in shared memory, no global traffic), to tell
// how close the warp-level instruction pattern alone gets to the DMMA peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gemm_micro tools/gemm_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// NW warps; warp tile (MI*8) x (NI*8); smem holds one BK=16 stage of a (WM*MI*8) x 16
// A tile and a 16 x (WN*NI*8) B tile in the kernel's padded layouts (k-major rows).
template <int MI, int NI, int WM, int WN, bool SYNC, int ORDER>
__global__ void __launch_bounds__(32 * WM * WN) loop(double* out, int iters) {
  constexpr int BM = WM * MI * 8, BN = WN * NI * 8, PAD = 4, BK = 16;
  __shared__ double As[BK * (BM + PAD)];
  __shared__ double Bs[BK * (BN + PAD)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, wm = warp % WM, wn = warp / WM;
  for (int i = tid; i < BK * (BM + PAD); i += blockDim.x) As[i] = 1e-3 * (i % 97);
  for (int i = tid; i < BK * (BN + PAD); i += blockDim.x) Bs[i] = 1e-3 * (i % 89);
  __syncthreads();
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    if (SYNC) __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int k = kk * 4 + t;
      double a[MI], b[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[mi] = As[k * (BM + PAD) + wm * MI * 8 + mi * 8 + g];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = Bs[k * (BN + PAD) + wn * NI * 8 + ni * 8 + g];
      if (ORDER == 0) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma884(acc[mi][ni], b[ni], a[mi]);
      } else {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) dmma884(acc[mi][ni], a[mi], b[ni]);
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[tid] = s;
}

template <int MI, int NI, int WM, int WN, bool SYNC, int ORDER>
int run(const char* name, int occ, double* out) {
  const int iters = 20000, nw = WM * WN;
  const int blocks = 148 * occ;
  loop<MI, NI, WM, WN, SYNC, ORDER><<<blocks, 32 * nw>>>(out, 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    loop<MI, NI, WM, WN, SYNC, ORDER><<<blocks, 32 * nw>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 256 * 4 * MI * NI * (double)nw * blocks * iters;  // 4 kk per it
  printf("{\"variant\": \"%s\", \"occ\": %d, \"tflops\": %.2f}\n", name, occ, flops / (best * 1e-3) / 1e12);
  return 0;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  run<4, 4, 2, 2, false, 0>("32x32 warp, 4 warps, no sync, ord0", 3, out);
  run<4, 4, 2, 2, true, 0>("32x32 warp, 4 warps, sync/16k, ord0", 3, out);
  run<4, 4, 2, 2, false, 1>("32x32 warp, 4 warps, no sync, ord1", 3, out);
  run<4, 4, 4, 2, false, 0>("32x32 warp, 8 warps, no sync", 2, out);
  run<4, 4, 4, 2, true, 0>("32x32 warp, 8 warps, sync/16k", 2, out);
  run<8, 4, 2, 2, false, 0>("64x32 warp, 4 warps, no sync", 2, out);
  run<8, 4, 2, 2, true, 0>("64x32 warp, 4 warps, sync", 2, out);
  run<4, 4, 2, 2, false, 0>("32x32 warp, 4 warps, no sync, occ4", 4, out);
  run<2, 4, 2, 2, false, 0>("16x32 warp, 4 warps, no sync", 4, out);
  return 0;
}
