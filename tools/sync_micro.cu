// Barrier-latency microbenchmark (tuning tool, not part of the library): the
// per-column cost floor of the panel-QR leaf.  grid.sync() of a cooperative
// grid vs barrier.cluster of a thread-block cluster vs __syncthreads, and a
// global-memory round trip (write + grid.sync + read of G records).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sync_micro tools/sync_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_grid(int iters, double* buf, int G) {
  cg::grid_group grid = cg::this_grid();
  double s = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 33) buf[((i & 1) * G + blockIdx.x) * 33 + threadIdx.x] = i + threadIdx.x;
    grid.sync();
    for (int e = threadIdx.x; e < G * 33; e += blockDim.x) s += buf[(i & 1) * G * 33 + e];
    __syncthreads();
  }
  if (s == -1.0) buf[0] = s;
}

__global__ void k_gridonly(int iters) {
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < iters; ++i) grid.sync();
}

__global__ void k_cluster(int iters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double rec[64];
  double s = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 33) rec[threadIdx.x] = i + threadIdx.x;
    cl.sync();
    const int n = cl.num_blocks();
    for (int e = threadIdx.x; e < n * 33; e += blockDim.x) {
      const double* r = cl.map_shared_rank(rec, e / 33);
      s += r[e % 33];
    }
    cl.sync();
  }
  if (s == -1.0) out[0] = s;
}

__global__ void k_block(int iters, double* out) {
  __shared__ double x[256];
  double s = 0.0;
  for (int i = 0; i < iters; ++i) {
    x[threadIdx.x] = i;
    __syncthreads();
    s += x[(threadIdx.x + 1) & 255];
    __syncthreads();
  }
  if (s == -1.0) out[0] = s;
}

int main() {
  double* buf;
  cudaMalloc(&buf, 1 << 22);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int G : {8, 16, 64, 128}) {
    int it = iters;
    void* args[] = {&it};
    cudaLaunchCooperativeKernel((void*)k_gridonly, G, 256, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_gridonly, G, 256, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"barrier\": \"grid.sync\", \"ctas\": %d, \"us\": %.3f}\n", G, ms * 1e3 / iters);
    void* args2[] = {&it, &buf, &G};
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_grid, G, 256, args2, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"barrier\": \"write+grid.sync+read G records\", \"ctas\": %d, \"us\": %.3f}\n", G, ms * 1e3 / iters);
  }
  for (int C : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (C > 8) cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, k_cluster, iters, buf);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k_cluster, iters, buf);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"barrier\": \"2x cluster.sync + DSMEM read\", \"ctas\": %d, \"us\": %.3f, \"err\": \"%s\"}\n", C,
           ms * 1e3 / iters, cudaGetErrorString(err));
  }
  cudaEventRecord(e0);
  k_block<<<1, 256>>>(iters, buf);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"barrier\": \"2x __syncthreads\", \"ctas\": 1, \"us\": %.3f}\n", ms * 1e3 / iters);
  printf("{\"last_error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
