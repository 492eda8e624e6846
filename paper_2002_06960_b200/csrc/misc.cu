// Small HBM-bound helpers of the randUTV loop:
//   U := I, V := I
//   Keep_upper_triang / Set_to_zero of the factored column block
//   T11 := diag(D) after the small SVD
//   ||T(k:m, k:n)||_F for the truncated variant      (O11)
//   NaN/Inf pre-scan (RANDUTV_CHECK_FINITE)
// Grid-stride, coalesced along columns; the norm is a fixed-order two-pass
// reduction (deterministic).
#include "common.cuh"

namespace rutv {

namespace {

inline unsigned blocks_for(const Launch& L, i64 total, int threads = 256) {
  i64 b = (total + threads - 1) / threads;
  const i64 cap = (i64)L.device_sms * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

__global__ void set_identity_kernel(i64 rows, i64 cols, double* X, i64 ldx) {
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    X[r + c * ldx] = (r == c) ? 1.0 : 0.0;
  }
}

__global__ void set_identity_shift_kernel(i64 rows, i64 cols, i64 shift, double* X, i64 ldx) {
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    X[r + c * ldx] = (r - c == shift) ? 1.0 : 0.0;
  }
}

__global__ void copy_kernel(i64 rows, i64 cols, const double* __restrict__ S, i64 lds, double* __restrict__ D,
                            i64 ldd) {
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    D[r + c * ldd] = S[r + c * lds];
  }
}

__global__ void fill_kernel(i64 rows, i64 cols, double v, double* X, i64 ldx) {
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    X[r + c * ldx] = v;
  }
}

__global__ void triu_kernel(i64 rows, i64 cols, double* X, i64 ldx) {
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    if (r > c) X[r + c * ldx] = 0.0;
  }
}

__global__ void set_diag_kernel(i64 w, const double* __restrict__ d, double* X, i64 ldx) {
  const i64 total = w * w;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % w, c = i / w;
    X[r + c * ldx] = (r == c) ? d[r] : 0.0;
  }
}

constexpr int RED_BLOCKS = 512;

__global__ void sumsq_partial_kernel(i64 rows, i64 cols, const double* __restrict__ X, i64 ldx,
                                     double* __restrict__ partial) {
  __shared__ double red[8];
  const i64 total = rows * cols;
  double s = 0.0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    const double v = X[r + c * ldx];
    s += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += red[k];
    partial[blockIdx.x] = t;
  }
}

__global__ void sumsq_final_kernel(int n, const double* __restrict__ partial, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += partial[i];
    out[0] = t;
  }
}

__global__ void nonfinite_kernel(i64 rows, i64 cols, const double* __restrict__ X, i64 ldx, int* flag) {
  const i64 total = rows * cols;
  int bad = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = i % rows, c = i / rows;
    bad |= !isfinite(X[r + c * ldx]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

}  // namespace

#define RUTV_GRID_LAUNCH(kernel, total, ...)                          \
  do {                                                                \
    if ((total) <= 0) return 0;                                       \
    kernel<<<blocks_for(L, (total)), 256, 0, L.stream>>>(__VA_ARGS__); \
    L.count();                                                        \
    RUTV_CHECK_LAUNCH(#kernel);                                       \
    return 0;                                                         \
  } while (0)

int launch_set_identity(const Launch& L, i64 rows, i64 cols, double* X, i64 ldx) {
  RUTV_GRID_LAUNCH(set_identity_kernel, rows * cols, rows, cols, X, ldx);
}
int launch_set_identity_shift(const Launch& L, i64 rows, i64 cols, i64 shift, double* X, i64 ldx) {
  RUTV_GRID_LAUNCH(set_identity_shift_kernel, rows * cols, rows, cols, shift, X, ldx);
}
int launch_copy(const Launch& L, i64 rows, i64 cols, const double* S, i64 lds, double* D, i64 ldd) {
  RUTV_GRID_LAUNCH(copy_kernel, rows * cols, rows, cols, S, lds, D, ldd);
}
int launch_fill(const Launch& L, i64 rows, i64 cols, double v, double* X, i64 ldx) {
  RUTV_GRID_LAUNCH(fill_kernel, rows * cols, rows, cols, v, X, ldx);
}
int launch_triu(const Launch& L, i64 rows, i64 cols, double* X, i64 ldx) {
  RUTV_GRID_LAUNCH(triu_kernel, rows * cols, rows, cols, X, ldx);
}
int launch_set_diag(const Launch& L, i64 w, const double* d, double* X, i64 ldx) {
  RUTV_GRID_LAUNCH(set_diag_kernel, w * w, w, d, X, ldx);
}
int launch_nonfinite(const Launch& L, i64 rows, i64 cols, const double* X, i64 ldx, int* flag) {
  RUTV_GRID_LAUNCH(nonfinite_kernel, rows * cols, rows, cols, X, ldx, flag);
}

int launch_sumsq(const Launch& L, i64 rows, i64 cols, const double* X, i64 ldx, double* partial, double* out) {
  if (rows <= 0 || cols <= 0) {
    RUTV_CUDA(cudaMemsetAsync(out, 0, sizeof(double), L.stream));
    return 0;
  }
  sumsq_partial_kernel<<<RED_BLOCKS, 256, 0, L.stream>>>(rows, cols, X, ldx, partial);
  L.count();
  sumsq_final_kernel<<<1, 32, 0, L.stream>>>(RED_BLOCKS, partial, out);
  L.count();
  RUTV_CHECK_LAUNCH("sumsq");
  return 0;
}

}  // namespace rutv
