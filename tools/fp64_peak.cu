// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Measures the roofline denominator SURVEY.md §8(d) M4 asks for (FP64 peak is not
// in MEASURED_PEAKS.json). Prints one JSON line. Not part of the product library.
#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int NACC>
__global__ void __launch_bounds__(256) dmma884_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void __launch_bounds__(256) dmma16816_loop(double* out, int iters, double seed) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + (threadIdx.x + i) * 1e-3;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed - (threadIdx.x + i) * 1e-3;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <typename K>
static double time_kernel(K kern, int grid, int block, double* out, int iters, int reps, float* ms_out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters, 1.0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  *ms_out = best;
  return best;
}

// sustained: back-to-back launches for ~secs seconds
template <typename K>
static double sustained(K kern, int grid, int block, double* out, int iters, double secs, int* nlaunch) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  auto t0 = std::chrono::steady_clock::now();
  int n = 0;
  while (true) {
    for (int j = 0; j < 8; ++j) { kern<<<grid, block>>>(out, iters, 1.0); ++n; }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > secs) break;
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  *nlaunch = n;
  return ms;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
  const int block = 256, iters = 4096;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  // DMMA m8n8k4: 256 FMA per warp-instruction = 512 flop
  for (int occ : {1, 2, 4}) {
    int grid = sms * occ; float ms;
    time_kernel(dmma884_loop<8>, grid, block, out, iters, 5, &ms);
    double flops = 512.0 * 8 * iters * (double)grid * (block / 32);
    printf(", \"dmma884_occ%d_tflops\": %.3f", occ, flops / (ms * 1e-3) / 1e12);
  }
  for (int occ : {1, 2}) {
    int grid = sms * occ; float ms;
    time_kernel(dmma16816_loop<4>, grid, block, out, iters / 4, 5, &ms);
    double flops = 2.0 * 16 * 8 * 16 * 4 * (iters / 4) * (double)grid * (block / 32);
    printf(", \"dmma16816_occ%d_tflops\": %.3f", occ, flops / (ms * 1e-3) / 1e12);
  }
  for (int occ : {1, 2, 4}) {
    int grid = sms * occ; float ms;
    time_kernel(dfma_loop<8>, grid, block, out, iters, 5, &ms);
    double flops = 2.0 * 8 * iters * (double)grid * block;
    printf(", \"dfma_occ%d_tflops\": %.3f", occ, flops / (ms * 1e-3) / 1e12);
  }
  {
    int grid = sms * 2, n; double ms = sustained(dmma884_loop<8>, grid, block, out, iters, 4.0, &n);
    double flops = 512.0 * 8 * iters * (double)grid * (block / 32) * n;
    printf(", \"dmma884_sustained_tflops\": %.3f, \"sustained_s\": %.2f", flops / (ms * 1e-3) / 1e12, ms * 1e-3);
  }
  {
    int grid = sms * 2, n; double ms = sustained(dfma_loop<8>, grid, block, out, iters, 4.0, &n);
    double flops = 2.0 * 8 * iters * (double)grid * block * n;
    printf(", \"dfma_sustained_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
