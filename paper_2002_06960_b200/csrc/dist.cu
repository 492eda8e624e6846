// Column-sharded multi-GPU randUTV and its C ABI.
//
// The paper has no distributed algorithm (its parallelism is shared-memory
// tasks over disk-resident blocks); the sharding here
// follows from the structure of one randUTV step (Sec. 3.1): every
// O(r s b) product of a step splits by columns of the trailing matrix, so
//
//   A (and the working T) : 1-D block-cyclic by column blocks of width b,
//                           global block j on rank j mod P (load balance as the
//                           trailing matrix shrinks);
//   U, V                  : contiguous row ranges (every update of U and V is a
//                           right multiplication, P:1338-1340, P:1352-1354,
//                           P:1361-1362, hence row-local).
//
// Per sampled step i (k = i b, r = m - k, s = n - k, owner o = i mod P), with
// A_p the rank's trailing columns:
//   S1  G                   generated redundantly (same Philox counters)
//   S2  Y_p = A_p^T G        local rows of Y
//   S3  Z = sum_p A_p Y_p    AllReduce (r x b);  Y_p = A_p^T Z  local
//   S4  Y = AllGather(Y_p)   then the same deterministic QR(Y) on every rank
//   S5  X W = sum_p A_p W_p  AllReduce (m x b); A_p -= (X W) T_V W_p^T local;
//       V rows: local (every rank holds all of W_V)
//   S6  QR of column block i on its owner; Broadcast (W_U, T_U)
//   S7  A_p -= W_U T_U^T W_U^T A_p local;  U rows local
//   S8  Jacobi SVD on the owner; Broadcast (U_s, V_s) on the side communicator
//   S9  folds: owner T11 = diag d, A01 V_s; every rank U_s^T A12 (its
//       columns), U(:, blk) U_s, V(:, blk) V_s
// The S8/S9 overlap of the single-GPU driver is kept: they run on the side
// stream with their own communicator (split from the main one), in the same
// program order on every rank.
//
// Two communicator back ends implement the same four collectives:
//   * NCCL (libnccl.so.2, loaded at run time; torch's bundled copy), one
//     process per GPU, bootstrapped from an ncclUniqueId the caller
//     distributes (the Python layer uses torch.distributed);
//   * loopback: P virtual ranks as P host threads in one process on one GPU,
//     collectives done by device copies/sums between host barriers (no kernel
//     ever waits on another rank's kernel).  It runs the SAME SPMD driver and
//     is how the sharded path is parity-tested on a single GPU.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include <nccl.h>

#include "driver.cuh"

#ifndef RUTV_NCCL_PATH
#define RUTV_NCCL_PATH "libnccl.so.2"
#endif

namespace rutv {

void comm_free(Comm* c) { delete c; }
int comm_sync(Comm* c, cudaStream_t s) { return c->sync(s); }

// ---------------------------------------------------------------- NCCL

struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId;
  decltype(&ncclCommInitRank) CommInitRank;
  decltype(&ncclCommSplit) CommSplit;
  decltype(&ncclCommDestroy) CommDestroy;
  decltype(&ncclAllReduce) AllReduce;
  decltype(&ncclAllGather) AllGather;
  decltype(&ncclBroadcast) Broadcast;
  decltype(&ncclGetErrorString) GetErrorString;
  decltype(&ncclCommGetAsyncError) GetAsyncError;
  decltype(&ncclCommAbort) CommAbort;
};

static std::mutex g_nccl_mu;
static NcclApi g_nccl;

static char g_nccl_err[256] = "";

const NcclApi* nccl_api() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.ok) return &g_nccl;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen(RUTV_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "dlopen(libnccl.so.2): %s", dlerror());
    return nullptr;
  }
#define RUTV_SYM(field, name)                                              \
  g_nccl.field = (decltype(g_nccl.field))dlsym(h, name);                   \
  if (!g_nccl.field) {                                                     \
    snprintf(g_nccl_err, sizeof(g_nccl_err), "dlsym(%s) failed", name);    \
    return nullptr;                                                        \
  }
  RUTV_SYM(GetUniqueId, "ncclGetUniqueId");
  RUTV_SYM(CommInitRank, "ncclCommInitRank");
  RUTV_SYM(CommSplit, "ncclCommSplit");
  RUTV_SYM(CommDestroy, "ncclCommDestroy");
  RUTV_SYM(AllReduce, "ncclAllReduce");
  RUTV_SYM(AllGather, "ncclAllGather");
  RUTV_SYM(Broadcast, "ncclBroadcast");
  RUTV_SYM(GetErrorString, "ncclGetErrorString");
  RUTV_SYM(GetAsyncError, "ncclCommGetAsyncError");
  RUTV_SYM(CommAbort, "ncclCommAbort");
#undef RUTV_SYM
  g_nccl.ok = true;
  return &g_nccl;
}

#define RUTV_NCCL(call)                                                                      \
  do {                                                                                       \
    ncclResult_t r__ = (call);                                                               \
    if (r__ != ncclSuccess) {                                                                \
      snprintf(g_nccl_err, sizeof(g_nccl_err), "%s: %s", #call, api->GetErrorString(r__));   \
      ::rutv::set_last_error(g_nccl_err, cudaErrorUnknown);                                  \
      return RANDUTV_ERR_NCCL;                                                               \
    }                                                                                        \
  } while (0)

// RUTV_NCCL_TIMEOUT_S: seconds a sharded call may wait on its collectives
// before aborting the communicator (default 1800; <= 0 waits forever)
static double nccl_timeout_s() {
  static double t = -1.0;
  if (t < 0.0) {
    const char* e = getenv("RUTV_NCCL_TIMEOUT_S");
    t = e ? atof(e) : 1800.0;
    if (t < 0.0) t = 0.0;
  }
  return t;
}

struct NcclComm : Comm {
  const NcclApi* api;
  ncclComm_t comm = nullptr;
  NcclComm* partner = nullptr;  // the side-stream communicator split from this one
  ~NcclComm() override {
    if (comm) api->CommDestroy(comm);
  }
  // abort this communicator and its partner: a collective of either may be
  // the one stuck on a dead peer
  void abort_all() {
    if (comm) api->CommAbort(comm);
    comm = nullptr;
    if (partner && partner->comm) {
      api->CommAbort(partner->comm);
      partner->comm = nullptr;
    }
  }
  int sync(cudaStream_t s) override {
    const double limit = nccl_timeout_s();
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) return 0;
      if (q != cudaErrorNotReady) {
        ::rutv::set_last_error("cudaStreamQuery (sharded call)", q);
        return RANDUTV_ERR_CUDA;
      }
      ncclResult_t ae = ncclSuccess;
      if (api->GetAsyncError(comm, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
        snprintf(g_nccl_err, sizeof(g_nccl_err), "NCCL asynchronous error: %s (communicator aborted)",
                 api->GetErrorString(ae));
        ::rutv::set_last_error(g_nccl_err, cudaErrorUnknown);
        abort_all();
        return RANDUTV_ERR_NCCL;
      }
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (limit > 0.0 && el > limit) {
        snprintf(g_nccl_err, sizeof(g_nccl_err),
                 "sharded call still waiting on its collectives after %.0f s (RUTV_NCCL_TIMEOUT_S): "
                 "communicator aborted", el);
        ::rutv::set_last_error(g_nccl_err, cudaErrorUnknown);
        abort_all();
        return RANDUTV_ERR_NCCL;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(el < 0.01 ? 20 : 500));
    }
  }
  int allreduce_sum(double* buf, i64 count, cudaStream_t s) override {
    if (count <= 0) return 0;
    if (!comm) return RANDUTV_ERR_NCCL;
    RUTV_NCCL(api->AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, comm, s));
    return 0;
  }
  int allgather(const double* send, double* recv, i64 count, cudaStream_t s) override {
    if (count <= 0) return 0;
    if (!comm) return RANDUTV_ERR_NCCL;
    RUTV_NCCL(api->AllGather(send, recv, (size_t)count, ncclFloat64, comm, s));
    return 0;
  }
  int bcast(double* buf, i64 count, int root, cudaStream_t s) override {
    if (count <= 0) return 0;
    if (!comm) return RANDUTV_ERR_NCCL;
    RUTV_NCCL(api->Broadcast(buf, buf, (size_t)count, ncclFloat64, root, comm, s));
    return 0;
  }
  int allreduce_min_int(int* buf, i64 count, cudaStream_t s) override {
    if (count <= 0) return 0;
    if (!comm) return RANDUTV_ERR_NCCL;
    RUTV_NCCL(api->AllReduce(buf, buf, (size_t)count, ncclInt32, ncclMin, comm, s));
    return 0;
  }
  int chunks() const override { return nranks > 1 ? 4 : 1; }
  bool capturable() const override { return true; }
};

// ---------------------------------------------------------------- loopback

constexpr int kMaxLoopRanks = 16;

struct PtrPack {
  const double* p[kMaxLoopRanks];
};

__global__ void sum_ranks_kernel(i64 count, int P, PtrPack src, double* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < count; i += (i64)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += src.p[q][i];  // fixed rank order: identical on every rank
    out[i] = s;
  }
}

struct LoopShared {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const void*> ptr;
  explicit LoopShared(int P_) : P(P_), ptr(P_, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LoopComm : Comm {
  LoopShared* sh;
  double* tmp = nullptr;  // per-rank reduction target
  i64 tmp_elems = 0;
  int sms = 148;
  ~LoopComm() override {
    if (tmp) cudaFree(tmp);
  }
  int grow(i64 elems) {
    if (elems <= tmp_elems) return 0;
    if (tmp) cudaFree(tmp);
    tmp = nullptr;
    tmp_elems = 0;
    RUTV_CUDA(cudaMalloc(&tmp, (size_t)elems * sizeof(double)));
    tmp_elems = elems;
    return 0;
  }
  // publish `p`, wait until every rank has published and drained its stream
  int publish(const void* p, cudaStream_t s) {
    RUTV_CUDA(cudaStreamSynchronize(s));
    sh->ptr[rank] = p;
    sh->barrier();
    return 0;
  }
  int allreduce_sum(double* buf, i64 count, cudaStream_t s) override {
    if (count <= 0) return 0;
    int st = grow(count);
    RUTV_TRY(publish(buf, s));
    if (st == 0) {
      PtrPack pk{};
      for (int q = 0; q < nranks; ++q) pk.p[q] = (const double*)sh->ptr[q];
      i64 blocks = std::min<i64>((count + 255) / 256, (i64)sms * 8);
      sum_ranks_kernel<<<(unsigned)blocks, 256, 0, s>>>(count, nranks, pk, tmp);
      if (cudaStreamSynchronize(s) != cudaSuccess) st = RANDUTV_ERR_CUDA;
    }
    sh->barrier();  // every rank has read every buffer
    if (st == 0 && cudaMemcpyAsync(buf, tmp, (size_t)count * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      st = RANDUTV_ERR_CUDA;
    if (st == 0 && cudaStreamSynchronize(s) != cudaSuccess) st = RANDUTV_ERR_CUDA;
    sh->barrier();
    return st;
  }
  int allgather(const double* send, double* recv, i64 count, cudaStream_t s) override {
    if (count <= 0) return 0;
    RUTV_TRY(publish(send, s));
    int st = 0;
    for (int q = 0; q < nranks && st == 0; ++q)
      if (cudaMemcpyAsync(recv + (i64)q * count, sh->ptr[q], (size_t)count * 8, cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess)
        st = RANDUTV_ERR_CUDA;
    if (st == 0 && cudaStreamSynchronize(s) != cudaSuccess) st = RANDUTV_ERR_CUDA;
    sh->barrier();
    return st;
  }
  int bcast(double* buf, i64 count, int root, cudaStream_t s) override {
    if (count <= 0) return 0;
    RUTV_TRY(publish(buf, s));
    int st = 0;
    if (rank != root) {
      if (cudaMemcpyAsync(buf, sh->ptr[root], (size_t)count * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        st = RANDUTV_ERR_CUDA;
    }
    sh->barrier();
    return st;
  }
  int allreduce_min_int(int* buf, i64 count, cudaStream_t s) override {
    if (count <= 0) return 0;
    RUTV_TRY(publish(buf, s));
    std::vector<int> acc((size_t)count, 0x7fffffff), h((size_t)count);
    int st = 0;
    for (int q = 0; q < nranks && st == 0; ++q) {
      if (cudaMemcpy(h.data(), sh->ptr[q], (size_t)count * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
        st = RANDUTV_ERR_CUDA;
        break;
      }
      for (i64 e = 0; e < count; ++e) acc[e] = std::min(acc[e], h[e]);
    }
    sh->barrier();
    if (st == 0 && cudaMemcpy(buf, acc.data(), (size_t)count * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      st = RANDUTV_ERR_CUDA;
    sh->barrier();
    return st;
  }
};

// ============================================================== layout kernels

// Y(0:s, 0:cols) in global trailing-column order from the all-gathered local
// chunks (rank q's chunk at Yall + q*stride, ld ldc, rows = q's trailing
// columns in local order).
__global__ void cyclic_gather_rows_kernel(i64 s, i64 cols, i64 k, i64 b, int P, i64 i, const double* __restrict__ Yall,
                                          i64 ldc, i64 stride, double* __restrict__ Y, i64 ldy) {
  const i64 total = s * cols;
  for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
    const i64 t = idx % s, col = idx / s;
    const i64 c = k + t, j = c / b;
    const int q = (int)(j % P);
    const i64 lb0 = i > q ? (i - q + P - 1) / P : 0;
    const i64 lr = (j / P - lb0) * b + c % b;
    Y[t + col * ldy] = Yall[q * stride + lr + col * ldc];
  }
}

// Wl(0:sl, 0:cols) = the rows of W (global trailing order, ld ldw) that belong
// to rank p's trailing columns.
__global__ void cyclic_scatter_rows_kernel(i64 sl, i64 cols, i64 k, i64 b, int P, int p, i64 lb0,
                                           const double* __restrict__ W, i64 ldw, double* __restrict__ Wl, i64 ldl) {
  const i64 total = sl * cols;
  for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
    const i64 lr = idx % sl, col = idx / sl;
    const i64 j = (lb0 + lr / b) * P + p;
    const i64 t = j * b + lr % b - k;
    Wl[lr + col * ldl] = W[t + col * ldw];
  }
}

// out[lc] = sum_{r >= k} X(r, lc)^2 for the local columns whose global index is
// >= k (0 otherwise): one CTA per column, fixed-order tree (deterministic)
__global__ void cyclic_colsumsq_kernel(i64 m, i64 nl, i64 k, i64 b, int P, int p, const double* __restrict__ X,
                                       i64 ldx, double* __restrict__ out) {
  __shared__ double red[256];
  for (i64 lc = blockIdx.x; lc < nl; lc += gridDim.x) {
    const i64 g = ((lc / b) * P + p) * b + lc % b;
    double acc = 0.0;
    if (g >= k)
      for (i64 r = k + threadIdx.x; r < m; r += blockDim.x) {
        const double v = X[r + lc * ldx];
        acc = fma(v, v, acc);
      }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[lc] = red[0];
    __syncthreads();
  }
}

__global__ void sum_vector_kernel(i64 cnt, const double* __restrict__ v, double* __restrict__ out) {
  __shared__ double red[256];
  double acc = 0.0;
  for (i64 i = threadIdx.x; i < cnt; i += blockDim.x) acc += v[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// launchers of the layout kernels for the host-streamed sharded driver (host.cu)
int launch_cyclic_gather_rows(const Launch& L, i64 s, i64 cols, i64 k, i64 b, int P, i64 i, const double* Yall,
                              i64 ldc, i64 stride, double* Y, i64 ldy);
int launch_cyclic_scatter_rows(const Launch& L, i64 sl, i64 cols, i64 k, i64 b, int P, int p, i64 lb0,
                               const double* W, i64 ldw, double* Wl, i64 ldl);

unsigned grid_for(const Launch& L, i64 total) {
  i64 b = (total + 255) / 256;
  const i64 cap = (i64)L.device_sms * 8;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

int launch_cyclic_gather_rows(const Launch& L, i64 s, i64 cols, i64 k, i64 b, int P, i64 i, const double* Yall,
                              i64 ldc, i64 stride, double* Y, i64 ldy) {
  if (s <= 0 || cols <= 0) return 0;
  cyclic_gather_rows_kernel<<<grid_for(L, s * cols), 256, 0, L.stream>>>(s, cols, k, b, P, i, Yall, ldc, stride, Y, ldy);
  L.count();
  RUTV_CHECK_LAUNCH("cyclic_gather_rows_kernel");
  return 0;
}

int launch_cyclic_scatter_rows(const Launch& L, i64 sl, i64 cols, i64 k, i64 b, int P, int p, i64 lb0,
                               const double* W, i64 ldw, double* Wl, i64 ldl) {
  if (sl <= 0 || cols <= 0) return 0;
  cyclic_scatter_rows_kernel<<<grid_for(L, sl * cols), 256, 0, L.stream>>>(sl, cols, k, b, P, p, lb0, W, ldw, Wl, ldl);
  L.count();
  RUTV_CHECK_LAUNCH("cyclic_scatter_rows_kernel");
  return 0;
}

// ============================================================== SPMD driver

struct DistWork {
  Work w;
  double *Yl, *Yall, *Wl, *wbuf, *svd;
  double* lefts;   // truncated: per step W_U (m x b, ld r), T_U (b x b), U_s (b x b)
  double* colss;   // truncated: per-local-column sums of squares (n_p), then the total
  double* blk;     // truncated: one row block of U_k (b x k) for the U_s application
  double* blkz;    // the pending row block's partial (T W_V) rows (b x b) for its AllReduce
  double* zc;      // chunked GEMM -> AllReduce: the row chunks, each contiguous (m x b)
};

size_t carve_dist(Carver& c, DistWork& d, const Layout& lay, i64 K, i64 k) {
  const i64 m = lay.m, n = lay.n, b = std::min(lay.b, lay.n);
  const i64 maxs = std::max<i64>(lay.max_trailing(0), 1);
  carve(c, d.w, m, n, b, 0, false);
  d.Yl = c.take<double>(maxs * b);
  d.Yall = c.take<double>((i64)lay.P * maxs * b);
  d.Wl = c.take<double>(maxs * b);
  d.wbuf = c.take<double>(m * b + b * b);
  d.svd = c.take<double>(2 * b * b);
  d.lefts = K > 0 ? c.take<double>(K * (m * b + 2 * b * b)) : nullptr;
  d.colss = K > 0 ? c.take<double>(lay.ncols(lay.p) + 8) : nullptr;
  d.blk = K > 0 ? c.take<double>(b * k) : nullptr;
  d.blkz = c.take<double>(b * b);
  d.zc = c.take<double>(m * b);
  return c.off;
}

struct DistProblem {
  Layout lay;
  int q;
  uint64_t seed;
  double* A;  // local columns, ld lda
  i64 lda;
  double* U;  // rows [u0, u0 + mu) of U (m x m), ld ldu; may be null
  i64 ldu, u0, mu;
  double* V;  // rows [v0, v0 + nv) of V (n x n), ld ldv; may be null
  i64 ldv, v0, nv;
  bool record;  // truncated with U_k: keep (W_U, T_U, U_s) of every step
  bool uv;      // U and V requested (rank-uniform; U / V above are null on ranks without rows)
};

constexpr int kMaxChunks = 4;

struct DistRun {
  randutv_ctx* ctx;
  Comm* comm;
  Comm* side_comm;
  DistWork d;
  DistProblem P;
  Launch L, S;
  // V stream (one CTA per GEMM tile, as the single-GPU driver): the V update of
  // step i after QR(Y) and the U update after the (W_U, T_U) broadcast run
  // there, overlapping the column-block QR, the T updates and the next step's
  // sampling; events: eWv / eV (W_V ready / V updated), eWu / eU (likewise U)
  Launch V;
  bool vs = false;
  cudaStream_t cs = nullptr;  // comm stream of the chunked main-stream AllReduces
};

// Z (rows x cols, ld ldz) := produce() then summed over the ranks, in row
// chunks: chunk c is produced into its own contiguous slice of R.d.zc (ld =
// its row count), AllReduced on the comm stream while the next chunk's GEMM
// runs on the main stream, and copied into Z.  `produce(r0, r1, dst, ldd)`
// enqueues the main-stream work for rows [r0, r1).
template <class F>
int gemm_allreduce_rows(DistRun& R, i64 rows, i64 cols, double* Z, i64 ldz, F&& produce) {
  const Launch& L = R.L;
  cudaStream_t st = L.stream;
  int nc = R.comm->chunks();
  if (nc > kMaxChunks) nc = kMaxChunks;
  if (rows < 64 * nc) nc = 1;
  if (nc == 1) {
    RUTV_TRY(produce(0, rows, Z, ldz));
    return R.comm->allreduce_sum(Z, rows * cols, st);  // (ldz == rows for the callers)
  }
  i64 off[kMaxChunks + 1];
  for (int c = 0; c <= nc; ++c) off[c] = rows * c / nc;
  for (int c = 0; c < nc; ++c) {
    const i64 rc = off[c + 1] - off[c];
    double* zc = R.d.zc + off[c] * cols;
    RUTV_TRY(produce(off[c], off[c + 1], zc, rc));
    RUTV_CUDA(cudaEventRecord(R.ctx->ecomm[c], st));
    RUTV_CUDA(cudaStreamWaitEvent(R.cs, R.ctx->ecomm[c], 0));
    RUTV_TRY(R.comm->allreduce_sum(zc, rc * cols, R.cs));
    RUTV_CUDA(cudaEventRecord(R.ctx->ecomm[kMaxChunks + c], R.cs));
  }
  for (int c = 0; c < nc; ++c) {
    const i64 rc = off[c + 1] - off[c];
    RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->ecomm[kMaxChunks + c], 0));
    RUTV_TRY(launch_copy(L, rc, cols, R.d.zc + off[c] * cols, rc, Z + off[c], ldz));
  }
  return 0;
}

// S8 + S9 of a block of width bw whose SVD the owner computes; runs on `Ls`
// with collectives on `cm`.
int dist_svd_and_fold(DistRun& R, const Launch& Ls, Comm* cm, i64 i, i64 bw, bool dense_final) {
  (void)dense_final;
  const Layout& lay = R.P.lay;
  const int p = lay.p, o = (int)(i % lay.P);
  const i64 k = i * lay.b;
  Work& w = R.d.w;
  double* Us = R.d.svd;
  double* Vs = R.d.svd + bw * bw;
  const i64 lc = (i / lay.P) * lay.b;  // owner's local column of block i
  if (p == o) {
    double* T11 = R.P.A + k + lc * R.P.lda;
    RUTV_TRY(launch_jacobi_svd(Ls, bw, T11, R.P.lda, Us, w.d, Vs, w.status, (int)(i + 1), w.jac, w.jac_elems));
  }
  RUTV_TRY(cm->bcast(R.d.svd, 2 * bw * bw, o, Ls.stream));
  if (R.P.record) {
    const i64 bb = lay.b, rec = i * (lay.m * bb + 2 * bb * bb);
    RUTV_CUDA(cudaMemcpyAsync(R.d.lefts + rec + (lay.m - k) * bb + bb * bb, Us, bw * bw * 8, cudaMemcpyDeviceToDevice,
                              Ls.stream));
  }
  if (p == o) {
    double* T11 = R.P.A + k + lc * R.P.lda;
    RUTV_TRY(launch_set_diag(Ls, bw, w.d, T11, R.P.lda));
    RUTV_TRY(right_mult_inplace(Ls, w.Zf, k, bw, R.P.A + lc * R.P.lda, R.P.lda, Vs, bw));  // A01 V_s
  }
  // U_s^T A12 over this rank's columns right of block i
  const i64 c1 = lay.lcol(p, i + 1);
  RUTV_TRY(left_mult_t_inplace(Ls, w.Zf, bw, lay.ncols(p) - c1, R.P.A + k + c1 * R.P.lda, R.P.lda, Us, bw));
  if (R.P.U) RUTV_TRY(right_mult_inplace(Ls, w.Zf, R.P.mu, bw, R.P.U + k * R.P.ldu, R.P.ldu, Us, bw));
  if (R.P.V) RUTV_TRY(right_mult_inplace(Ls, w.Zf, R.P.nv, bw, R.P.V + k * R.P.ldv, R.P.ldv, Vs, bw));
  return 0;
}

int dist_sampled_step(DistRun& R, i64 i) {
  const Layout& lay = R.P.lay;
  const Launch& L = R.L;
  Work& w = R.d.w;
  const int p = lay.p, P = lay.P, o = (int)(i % P);
  const i64 m = lay.m, n = lay.n, b = lay.b, k = i * b, r = m - k, s = n - k;
  const i64 c0 = lay.lcol(p, i), sl = lay.ncols(p) - c0, maxs = std::max<i64>(lay.max_trailing(i), 1);
  double* Ap = R.P.A + c0 * R.P.lda;  // this rank's trailing columns, all m rows
  double* At = Ap + k;                // rows k:m
  const i64 lda = R.P.lda;
  cudaStream_t st = L.stream;
  // S1, S2, S3
  RUTV_TRY(launch_gaussian(L, R.P.seed, i, r, b, w.G, r));
  RUTV_TRY(launch_dgemm(L, true, false, sl, b, r, 1.0, At, lda, w.G, r, 0.0, R.d.Yl, maxs, w.gemm_ws, w.gemm_ws_elems));
  for (int qq = 0; qq < R.P.q; ++qq) {
    // Z = sum_p A_p Y_p, pipelined in row chunks with its AllReduce
    RUTV_TRY(gemm_allreduce_rows(R, r, b, w.Z, r, [&](i64 r0, i64 r1, double* dst, i64 ldd) {
      return launch_dgemm(L, false, false, r1 - r0, b, sl, 1.0, At + r0, lda, R.d.Yl, maxs, 0.0, dst, ldd,
                          w.gemm_ws, w.gemm_ws_elems);
    }));
    RUTV_TRY(launch_dgemm(L, true, false, sl, b, r, 1.0, At, lda, w.Z, r, 0.0, R.d.Yl, maxs, w.gemm_ws,
                          w.gemm_ws_elems));
  }
  // S4: gather Y in global order, the same QR on every rank
  RUTV_TRY(R.comm->allgather(R.d.Yl, R.d.Yall, maxs * b, st));
  cyclic_gather_rows_kernel<<<grid_for(L, s * b), 256, 0, st>>>(s, b, k, b, P, i, R.d.Yall, maxs, maxs * b, w.Y, s);
  L.count();
  RUTV_CHECK_LAUNCH("cyclic_gather_rows_kernel");
  if (R.vs) RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->eV, 0));  // the previous V update read W_V, T_V
  RUTV_TRY(panel_qr(L, s, b, w.Y, s, w.tauV, w.Wv, s, w.TV, b, w.qw));
  // S5 for the V rows (every rank holds all of W_V; V is not touched by the
  // folds of T): on the V stream, overlapping the rest of the step
  if (R.P.V) {
    if (R.vs) {
      RUTV_CUDA(cudaEventRecord(R.ctx->eWv, st));
      RUTV_CUDA(cudaStreamWaitEvent(R.V.stream, R.ctx->eWv, 0));
      Work wv = w;
      wv.Z = w.Zv;
      wv.Z2 = w.Zv2;
      wv.gemm_ws = w.gemm_ws_v;
      wv.gemm_ws_elems = 4 * std::max(lay.m, lay.n) * b;
      RUTV_TRY(apply_right(R.V, wv, R.P.nv, s, b, R.P.V + k * R.P.ldv, R.P.ldv, w.Wv, s, w.TV, b));
    } else {
      RUTV_TRY(apply_right(L, w, R.P.nv, s, b, R.P.V + k * R.P.ldv, R.P.ldv, w.Wv, s, w.TV, b));
    }
  }
  if (R.vs) RUTV_CUDA(cudaEventRecord(R.ctx->eV, R.V.stream));
  const bool fuse = fuse_left();
  // Fused path: the side stream's folds of step i-1 write only row block i-1
  // (rows pk .. k) of the trailing columns, so every other row runs S5-S7
  // before waiting for them (the SVD of step i-1 hides behind the step) and the
  // pending rows get their S5 afterwards.  Unfused: wait first.
  const i64 pk = (fuse && k > 0) ? k - b : k, pb = k - pk;
  if (!fuse) RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->eF, 0));
  if (sl > 0) {
    cyclic_scatter_rows_kernel<<<grid_for(L, sl * b), 256, 0, st>>>(sl, b, k, b, P, p, lay.lb_before(p, i), w.Wv, s,
                                                                   R.d.Wl, maxs);
    L.count();
    RUTV_CHECK_LAUNCH("cyclic_scatter_rows_kernel");
  }
  // Z = T W_V (AllReduce, m x b; the pending rows are zero here and done
  // later), pipelined in row chunks with its AllReduce
  RUTV_TRY(gemm_allreduce_rows(R, m, b, w.Z, m, [&](i64 r0, i64 r1, double* dst, i64 ldd) {
    // rows [0, pk): T rows above the pending block; [pk, k): zero; [k, m): A_t
    const i64 a0 = std::max<i64>(r0, 0), a1 = std::min<i64>(r1, pk);
    if (a1 > a0)
      RUTV_TRY(launch_dgemm(L, false, false, a1 - a0, b, sl, 1.0, Ap + a0, lda, R.d.Wl, maxs, 0.0, dst + (a0 - r0),
                            ldd, w.gemm_ws, w.gemm_ws_elems));
    const i64 z0 = std::max<i64>(r0, pk), z1 = std::min<i64>(r1, k);
    if (z1 > z0) RUTV_TRY(launch_fill(L, z1 - z0, b, 0.0, dst + (z0 - r0), ldd));
    const i64 t0 = std::max<i64>(r0, k), t1 = std::min<i64>(r1, m);
    if (t1 > t0)
      RUTV_TRY(launch_dgemm(L, false, false, t1 - t0, b, sl, 1.0, Ap + t0, lda, R.d.Wl, maxs, 0.0, dst + (t0 - r0),
                            ldd, w.gemm_ws, w.gemm_ws_elems));
    return 0;
  }));
  RUTV_TRY(launch_dgemm(L, false, false, m, b, b, 1.0, w.Z, m, w.TV, b, 0.0, w.Z2, m, nullptr, 0));
  // S5 update: unfused -- every trailing column of every row; fused -- column
  // block i (its owner) for the rows outside the pending block
  const i64 ucols = fuse ? (p == o ? b : 0) : sl;
  if (pk > 0)
    RUTV_TRY(launch_dgemm(L, false, true, pk, ucols, b, -1.0, w.Z2, m, R.d.Wl, maxs, 1.0, Ap, lda, nullptr, 0));
  RUTV_TRY(launch_dgemm(L, false, true, m - pk - pb, ucols, b, -1.0, w.Z2 + k, m, R.d.Wl, maxs, 1.0, At, lda,
                        nullptr, 0));
  // S6: QR of column block i on its owner, broadcast (W_U, T_U)
  double* Wu = R.d.wbuf;
  double* TU = R.d.wbuf + r * b;
  if (p == o) {
    RUTV_TRY(panel_qr(L, r, b, At, lda, w.tauU, Wu, r, TU, b, w.qw));
    RUTV_TRY(launch_triu(L, b, b, At, lda));
    RUTV_TRY(launch_fill(L, r - b, b, 0.0, At + b, lda));
  }
  if (R.vs) RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->eU, 0));  // the previous U update read W_U, T_U
  RUTV_TRY(R.comm->bcast(R.d.wbuf, r * b + b * b, o, st));
  if (R.P.record) RUTV_CUDA(cudaMemcpyAsync(R.d.lefts + i * (m * b + 2 * b * b), R.d.wbuf, (r * b + b * b) * 8,
                                            cudaMemcpyDeviceToDevice, st));
  // S7 (fused with the rest of S5 when enabled): columns right of block i; U rows
  const i64 c1 = lay.lcol(p, i + 1);
  if (fuse)
    RUTV_TRY(fused_right_left(L, w, m, r, b, k, lay.ncols(p) - c1, R.P.A + c1 * lda, lda, R.d.Wl + (c1 - c0), maxs,
                              w.Z2, m, Wu, r, TU, b, pk));
  else
    RUTV_TRY(apply_left_t(L, w, r, lay.ncols(p) - c1, b, R.P.A + k + c1 * lda, lda, Wu, r, TU, b));
  if (R.P.U) {
    if (R.vs) {
      RUTV_CUDA(cudaEventRecord(R.ctx->eWu, st));
      RUTV_CUDA(cudaStreamWaitEvent(R.V.stream, R.ctx->eWu, 0));
      Work wu = w;
      wu.Z = w.Zv;
      wu.Z2 = w.Zv2;
      wu.gemm_ws = w.gemm_ws_v;
      wu.gemm_ws_elems = 4 * std::max(lay.m, lay.n) * b;
      RUTV_TRY(apply_right(R.V, wu, R.P.mu, r, b, R.P.U + k * R.P.ldu, R.P.ldu, Wu, r, TU, b));
    } else {
      RUTV_TRY(apply_right(L, w, R.P.mu, r, b, R.P.U + k * R.P.ldu, R.P.ldu, Wu, r, TU, b));
    }
  }
  if (R.vs) RUTV_CUDA(cudaEventRecord(R.ctx->eU, R.V.stream));
  if (fuse) {
    RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->eF, 0));
    if (pb > 0) {
      // S5 of the pending row block over all of this rank's trailing columns
      RUTV_TRY(launch_dgemm(L, false, false, pb, b, sl, 1.0, Ap + pk, lda, R.d.Wl, maxs, 0.0, w.Z + pk, m,
                            w.gemm_ws, w.gemm_ws_elems));
      RUTV_TRY(launch_copy(L, pb, b, w.Z + pk, m, R.d.blkz, pb));
      RUTV_TRY(R.comm->allreduce_sum(R.d.blkz, pb * b, st));
      RUTV_TRY(launch_dgemm(L, false, false, pb, b, b, 1.0, R.d.blkz, pb, w.TV, b, 0.0, w.Z2 + pk, m, nullptr, 0));
      RUTV_TRY(launch_dgemm(L, false, true, pb, sl, b, -1.0, w.Z2 + pk, m, R.d.Wl, maxs, 1.0, Ap + pk, lda, nullptr,
                            0));
    }
  }
  // S8, S9 on the side stream / side communicator
  RUTV_CUDA(cudaEventRecord(R.ctx->eR, st));
  RUTV_CUDA(cudaStreamWaitEvent(R.S.stream, R.ctx->eR, 0));
  if (R.vs) RUTV_CUDA(cudaStreamWaitEvent(R.S.stream, R.ctx->eU, 0));  // U(:, blk), V(:, blk) folds
  RUTV_TRY(dist_svd_and_fold(R, R.S, R.side_comm, i, b, false));
  RUTV_CUDA(cudaEventRecord(R.ctx->eF, R.S.stream));
  return 0;
}

int dist_final_step(DistRun& R, i64 i) {
  const Layout& lay = R.P.lay;
  const Launch& L = R.L;
  Work& w = R.d.w;
  const int p = lay.p, o = (int)(i % lay.P);
  const i64 m = lay.m, n = lay.n, k = i * lay.b, r = m - k, s = n - k;
  if (s <= 0) return 0;
  cudaStream_t st = L.stream;
  RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->eF, 0));
  if (R.vs) RUTV_CUDA(cudaStreamWaitEvent(st, R.ctx->eU, 0));  // eU follows eV on the V stream
  const i64 lc = (i / lay.P) * lay.b;
  double* At = R.P.A + k + lc * R.P.lda;
  if (r > s) {
    double* Wu = R.d.wbuf;
    double* TU = R.d.wbuf + r * s;
    if (p == o) {
      RUTV_TRY(panel_qr(L, r, s, At, R.P.lda, w.tauU, Wu, r, TU, s, w.qw));
      RUTV_TRY(launch_triu(L, s, s, At, R.P.lda));
      RUTV_TRY(launch_fill(L, r - s, s, 0.0, At + s, R.P.lda));
    }
    // participation in the broadcast depends on rank-uniform values only
    if (R.P.uv) RUTV_TRY(R.comm->bcast(R.d.wbuf, r * s + s * s, o, st));
    if (R.P.U) RUTV_TRY(apply_right(L, w, R.P.mu, r, s, R.P.U + k * R.P.ldu, R.P.ldu, Wu, r, TU, s));
  }
  return dist_svd_and_fold(R, L, R.comm, i, s, r == s);
}

// U_k = U(:, 0:k) of the truncated run by backward accumulation (reading A12)
// over this rank's rows [u0, u0 + mu): X := rows of [I_k; 0]; for j = K-1..0:
// X[kj:kj+b, kj:k] := U_s^(j) X[...] (the row block is gathered with an
// AllReduce of the ranks' disjoint rows), then X[kj:m, kj:k] -= W (T (W^T X))
// with W^T X summed over the ranks (AllReduce, b x (k - kj)).
int dist_backward_uk(DistRun& R, i64 K, i64 k) {
  const Layout& lay = R.P.lay;
  const Launch& L = R.L;
  Work& w = R.d.w;
  const i64 m = lay.m, b = lay.b, u0 = R.P.u0, mu = R.P.mu;
  double* X = R.P.U;
  const i64 ldx = R.P.ldu;
  cudaStream_t st = L.stream;
  RUTV_TRY(launch_set_identity_shift(L, mu, k, -u0, X, ldx));
  for (i64 j = K - 1; j >= 0; --j) {
    const i64 kj = j * b, rj = m - kj, cols = k - kj;
    const double* rec = R.d.lefts + j * (m * b + 2 * b * b);
    const double* Wj = rec;                   // rj x b, ld rj
    const double* Tj = rec + rj * b;          // b x b
    const double* Usj = rec + rj * b + b * b; // b x b
    // (a) rows kj..kj+b: gather, U_s, scatter back
    const i64 lo = std::max(u0, kj), hi = std::min(u0 + mu, kj + b);
    RUTV_TRY(launch_fill(L, b, cols, 0.0, R.d.blk, b));
    if (hi > lo) RUTV_TRY(launch_copy(L, hi - lo, cols, X + (lo - u0) + kj * ldx, ldx, R.d.blk + (lo - kj), b));
    RUTV_TRY(R.comm->allreduce_sum(R.d.blk, b * cols, st));
    if (hi > lo) {
      RUTV_TRY(launch_dgemm(L, false, false, b, cols, b, 1.0, Usj, b, R.d.blk, b, 0.0, w.Z, b, nullptr, 0));
      RUTV_TRY(launch_copy(L, hi - lo, cols, w.Z + (lo - kj), b, X + (lo - u0) + kj * ldx, ldx));
    }
    // (b) X[kj:m] -= W (T (W^T X[kj:m]))   (local rows >= kj)
    const i64 l0 = std::max(u0, kj), nrow = u0 + mu - l0;  // local rows in [kj, m)
    double* Xr = X + (l0 - u0) + kj * ldx;
    const double* Wr = Wj + (l0 - kj);
    RUTV_TRY(launch_dgemm(L, true, false, b, cols, nrow > 0 ? nrow : 0, 1.0, Wr, rj, Xr, ldx, 0.0, w.Z, b, w.gemm_ws,
                          w.gemm_ws_elems));
    RUTV_TRY(R.comm->allreduce_sum(w.Z, b * cols, st));
    RUTV_TRY(launch_dgemm(L, false, false, b, cols, b, 1.0, Tj, b, w.Z, b, 0.0, w.Z2, b, nullptr, 0));
    if (nrow > 0) RUTV_TRY(launch_dgemm(L, false, false, nrow, cols, b, -1.0, Wr, rj, w.Z2, b, 1.0, Xr, ldx, nullptr, 0));
  }
  return 0;
}

// finish() of the sharded path: the wait goes through the communicator
// (asynchronous-error polling and timeout, NcclComm::sync)
int dist_finish(DistRun& R) {
  randutv_ctx* ctx = R.ctx;
  int status = 0x7f7f7f7f;
  RUTV_CUDA(cudaMemcpyAsync(&status, R.d.w.status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RUTV_TRY(R.comm->sync(ctx->stream));
  RUTV_CUDA(cudaGetLastError());
  if (ctx->prof.on) ctx->prof.collect();
  return status != 0x7f7f7f7f ? status : 0;
}

// Agreement before the first collective of a sharded call: every rank
// contributes whether its own checks passed (argument checks, workspace,
// finiteness scan); the minimum decides for all, so either every rank enters
// the collectives or none does.  Returns 1 if every rank is ready.
int agree(Comm* comm, cudaStream_t s, bool ready, int* all_ready) {
  if (!comm->dflag) RUTV_CUDA(cudaMalloc(&comm->dflag, sizeof(int)));
  int h = ready ? 1 : 0;
  RUTV_CUDA(cudaMemcpyAsync(comm->dflag, &h, sizeof(int), cudaMemcpyHostToDevice, s));
  RUTV_TRY(comm->allreduce_min_int(comm->dflag, 1, s));
  RUTV_CUDA(cudaMemcpyAsync(&h, comm->dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  RUTV_TRY(comm->sync(s));
  *all_ready = h;
  return 0;
}

int dist_run_loop(DistRun& R, i64 nsamp, bool trunc);

// RANDUTV_ASYNC (full factorisation only): everything enqueued -- the status
// AllReduce included -- and no host synchronisation, so the call can be
// captured into a CUDA graph with the NCCL collectives; randutv_wait gives
// the status through the communicator
int dist_run_async(DistRun& R) {
  randutv_ctx* ctx = R.ctx;
  RUTV_TRY(start_status(ctx, R.d.w));
  RUTV_TRY(dist_run_loop(R, sampled_steps(R.P.lay.n, R.P.lay.b), false));
  RUTV_TRY(R.comm->allreduce_min_int(R.d.w.status, 1, R.L.stream));
  ctx->async_status = R.d.w.status;
  ctx->async_dist = true;
  ctx->ws_captured = true;
  return 0;
}

// K = -1: full factorisation; K >= 1: truncated after K sampled steps (rank k)
int dist_run(DistRun& R, i64 K, i64 k, double* resid_fro) {
  const Layout& lay = R.P.lay;
  randutv_ctx* ctx = R.ctx;
  Work& w = R.d.w;
  const Launch& L = R.L;
  const bool trunc = K >= 0;
  const i64 nsamp = trunc ? K : sampled_steps(lay.n, lay.b);
  RUTV_TRY(start_status(ctx, w));
  RUTV_TRY(dist_run_loop(R, nsamp, trunc));
  if (trunc) {
    // rho^2 = sum over ranks of ||T(k:m, local columns >= k)||_F^2
    const i64 nl = lay.ncols(lay.p);
    RUTV_CUDA(cudaMemsetAsync(R.d.colss + nl, 0, sizeof(double), L.stream));
    if (nl > 0) {
      cyclic_colsumsq_kernel<<<(unsigned)std::min<i64>(nl, (i64)L.device_sms * 8), 256, 0, L.stream>>>(
          lay.m, nl, k, lay.b, lay.P, lay.p, R.P.A, R.P.lda, R.d.colss);
      L.count();
      RUTV_CHECK_LAUNCH("cyclic_colsumsq_kernel");
      sum_vector_kernel<<<1, 256, 0, L.stream>>>(nl, R.d.colss, R.d.colss + nl);
      L.count();
      RUTV_CHECK_LAUNCH("sum_vector_kernel");
    }
    RUTV_TRY(R.comm->allreduce_sum(R.d.colss + nl, 1, L.stream));
    if (R.P.record) RUTV_TRY(dist_backward_uk(R, K, k));  // collective: every rank, even without rows
    double ss = 0.0;
    RUTV_CUDA(cudaMemcpyAsync(&ss, R.d.colss + nl, sizeof(double), cudaMemcpyDeviceToHost, L.stream));
    RUTV_TRY(R.comm->allreduce_min_int(w.status, 1, L.stream));
    const int st = dist_finish(R);
    *resid_fro = std::sqrt(ss);
    return st;
  }
  // every rank returns the first non-converged block (status word: min)
  RUTV_TRY(R.comm->allreduce_min_int(w.status, 1, L.stream));
  return dist_finish(R);
}

// U := I, V := I (rows of the rank), the steps, the final step (full only),
// and every stream joined back into the main one
int dist_run_loop(DistRun& R, i64 nsamp, bool trunc) {
  const Layout& lay = R.P.lay;
  randutv_ctx* ctx = R.ctx;
  const Launch& L = R.L;
  if (!trunc && R.P.U && R.P.mu > 0) {
    RUTV_TRY(launch_set_identity_shift(L, R.P.mu, lay.m, -R.P.u0, R.P.U, R.P.ldu));  // rows u0.. of I
  }
  if (R.P.V && R.P.nv > 0) {
    RUTV_TRY(launch_set_identity_shift(L, R.P.nv, lay.n, -R.P.v0, R.P.V, R.P.ldv));
  }
  // the side, V and comm streams start after the initialisation
  RUTV_CUDA(cudaEventRecord(ctx->eF, L.stream));
  RUTV_CUDA(cudaStreamWaitEvent(R.cs, ctx->eF, 0));
  if (R.vs) {
    RUTV_CUDA(cudaStreamWaitEvent(R.V.stream, ctx->eF, 0));
    RUTV_CUDA(cudaEventRecord(ctx->eV, R.V.stream));
    RUTV_CUDA(cudaEventRecord(ctx->eU, R.V.stream));
  }
  // (truncated: the U updates are replaced by the records; P.U is the U_k output)
  double* Uk = R.P.U;
  if (trunc) R.P.U = nullptr;
  for (i64 i = 0; i < nsamp; ++i) RUTV_TRY(dist_sampled_step(R, i));
  if (!trunc) RUTV_TRY(dist_final_step(R, nsamp));
  R.P.U = Uk;
  RUTV_CUDA(cudaStreamWaitEvent(L.stream, ctx->eF, 0));
  if (R.vs) RUTV_CUDA(cudaStreamWaitEvent(L.stream, ctx->eU, 0));
  // the comm stream's last chunk was already waited for by the main stream
  // (gemm_allreduce_rows); join it anyway so a captured graph closes over it
  RUTV_CUDA(cudaEventRecord(ctx->ecomm[2 * kMaxChunks - 1], R.cs));
  RUTV_CUDA(cudaStreamWaitEvent(L.stream, ctx->ecomm[2 * kMaxChunks - 1], 0));
  return 0;
}

// argument checks shared by the NCCL and loopback entries; returns 0 or -i
// (positions of randutv_factor_dist)
int dist_check(const Layout& lay, const double* A, i64 lda, int q, unsigned flags, const double* U, i64 ldu,
               const double* V, i64 ldv) {
  const bool uv = !(flags & RANDUTV_NO_UV);
  if (flags & RANDUTV_REORTH) return -9;  // not implemented on the sharded path
  if (lay.n < 1) return -3;
  if (lay.m < lay.n) return -2;
  const i64 nc = lay.ncols(lay.p);
  if (nc > 0 && !A) return -4;
  if (lda < std::max<i64>(lay.m, 1)) return -5;
  if (lay.b < 1) return -6;
  if (q < 0) return -7;
  const i64 mu = Layout::row0(lay.m, lay.P, lay.p + 1) - Layout::row0(lay.m, lay.P, lay.p);
  const i64 nv = Layout::row0(lay.n, lay.P, lay.p + 1) - Layout::row0(lay.n, lay.P, lay.p);
  if (uv && mu > 0 && !U) return -10;
  if (uv && ldu < std::max<i64>(mu, 1)) return -11;
  if (uv && nv > 0 && !V) return -12;
  if (uv && ldv < std::max<i64>(nv, 1)) return -13;
  return 0;
}

// k == 0: full factorisation (U_local: rows of U, m x m); k >= 1: truncated
// rank-k (U_local: rows of U_k, m x k; *resid_fro = ||T(k:m, k:n)||_F)
int dist_factor(randutv_ctx* ctx, Comm* comm, Comm* side_comm, i64 m, i64 n, double* A, i64 lda, i64 b, int q,
                uint64_t seed, unsigned flags, double* U, i64 ldu, double* V, i64 ldv, i64 k, double* resid_fro) {
  Layout lay{m, n, std::max<i64>(1, std::min(b, n)), comm->nranks, comm->rank, 0};
  lay.nblocks = (n + lay.b - 1) / lay.b;
  // local checks first; no rank returns before the agreement, so a rank whose
  // arguments or workspace fail never leaves its peers blocked in a collective
  int local = b < 1 ? -6 : dist_check(lay, A, lda, q, flags, U, ldu, V, ldv);
  if (local == 0 && ctx->oversample > 0) local = -9;  // oversampling is single-GPU only
  if (local == 0 && fault_alloc(comm->rank)) {
    set_last_error("cudaMalloc(workspace) [RUTV_FAULT injected]", cudaErrorMemoryAllocation);
    local = RANDUTV_ERR_ALLOC;
  }
  const bool uv = !(flags & RANDUTV_NO_UV);
  i64 K = -1;
  if (local == 0 && k != 0) {
    K = (k + lay.b - 1) / lay.b;
    if (k < 0 || K > sampled_steps(n, lay.b)) local = -14;  // truncation needs k <= b * (sampled steps)
    else if (!resid_fro) local = -15;
  }
  DistRun R;
  R.ctx = ctx;
  R.comm = comm;
  R.side_comm = side_comm;
  R.L = ctx->launch();
  R.S = ctx->side_launch();
  R.V = ctx->v_launch();
  const bool async = (flags & RANDUTV_ASYNC) != 0;
  if (local == 0 && async && (!comm->capturable() || k != 0 || (flags & RANDUTV_CHECK_FINITE))) local = -9;
  if (local == 0 && !ctx->cstr) {
    if (cudaStreamCreateWithFlags(&ctx->cstr, cudaStreamNonBlocking) != cudaSuccess) local = RANDUTV_ERR_CUDA;
    for (int e = 0; e < 2 * kMaxChunks && local == 0; ++e)
      if (cudaEventCreateWithFlags(&ctx->ecomm[e], cudaEventDisableTiming) != cudaSuccess) local = RANDUTV_ERR_CUDA;
  }
  R.cs = ctx->cstr;
  if (local == 0) {
    Carver dry{nullptr, 0, 0, true};
    const size_t need = carve_dist(dry, R.d, lay, K > 0 ? K : 0, k);
    local = ensure_ws(ctx, need);
  }
  if (async) {
    // an ASYNC (graph-capturable) call cannot synchronise the host for the
    // agreement: the caller guarantees rank-uniform arguments, as NCCL itself
    // requires
    if (local != 0) return local;
  } else {
    int all = 0;
    RUTV_TRY(agree(comm, ctx->stream, local == 0, &all));
    if (local != 0) return local;
    if (!all) return RANDUTV_ERR_PEER;
  }
  Carver real{(char*)ctx->ws, 0, ctx->ws_bytes, false};
  carve_dist(real, R.d, lay, K > 0 ? K : 0, k);
  const i64 u0 = Layout::row0(m, lay.P, lay.p), u1 = Layout::row0(m, lay.P, lay.p + 1);
  const i64 v0 = Layout::row0(n, lay.P, lay.p), v1 = Layout::row0(n, lay.P, lay.p + 1);
  R.P = DistProblem{lay, q, seed, A, lda, uv ? U : nullptr, ldu, u0, u1 - u0, uv ? V : nullptr, ldv, v0, v1 - v0,
                    uv && K > 0, uv};
  if (R.P.U && R.P.mu == 0) R.P.U = nullptr;
  if (R.P.V && R.P.nv == 0) R.P.V = nullptr;
  {
    // RUTV_VSTREAM=0 keeps the U / V updates on the main stream (comparison only)
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("RUTV_VSTREAM");
      v = e ? atoi(e) : 1;
    }
    R.vs = uv && v != 0 && fuse_left();
  }
  if (flags & RANDUTV_CHECK_FINITE) {
    int bad = 0;
    if (lay.ncols(lay.p) > 0) bad = check_finite(ctx, R.L, R.d.w, m, lay.ncols(lay.p), A, lda);
    // agree on the verdict (a CUDA failure of the scan counts as "not clean")
    int all = 0;
    RUTV_TRY(agree(comm, ctx->stream, bad == 0, &all));
    if (bad != 0 && bad != RANDUTV_ERR_NONFINITE) return bad;
    if (!all) return RANDUTV_ERR_NONFINITE;
  }
  if (async) {
    RUTV_TRY(dist_run_async(R));
    ctx->stats.factorizations++;
    return 0;
  }
  const int st = dist_run(R, K, k, resid_fro);
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

}  // namespace rutv

// ============================================================================ C ABI

using namespace rutv;

extern "C" {

RANDUTV_API int randutv_dist_layout(int64_t m, int64_t n, int64_t b, int nranks, int rank, int64_t* out) {
  if (n < 1) return -2;
  if (m < n) return -1;
  if (b < 1) return -3;
  if (nranks < 1) return -4;
  if (rank < 0 || rank >= nranks) return -5;
  if (!out) return -6;
  const i64 bb = std::min<i64>(b, n);
  Layout lay{m, n, bb, nranks, rank, (n + bb - 1) / bb};
  out[0] = lay.ncols(rank);
  out[1] = Layout::row0(m, nranks, rank);
  out[2] = Layout::row0(m, nranks, rank + 1);
  out[3] = Layout::row0(n, nranks, rank);
  out[4] = Layout::row0(n, nranks, rank + 1);
  return 0;
}

RANDUTV_API int randutv_nccl_unique_id(void* out) {
  if (!out) return -1;
  const NcclApi* api = nccl_api();
  if (!api) {
    set_last_error(g_nccl_err, cudaErrorUnknown);
    return RANDUTV_ERR_NCCL;
  }
  ncclUniqueId id;
  RUTV_NCCL(api->GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return 0;
}

RANDUTV_API int randutv_comm_init(randutv_ctx* ctx, const void* unique_id, int nranks, int rank) {
  RUTV_TRY(begin_call(ctx));
  if (!unique_id) return -2;
  if (nranks < 1) return -3;
  if (rank < 0 || rank >= nranks) return -4;
  const NcclApi* api = nccl_api();
  if (!api) {
    set_last_error(g_nccl_err, cudaErrorUnknown);
    return RANDUTV_ERR_NCCL;
  }
  comm_free(ctx->comm_side);
  comm_free(ctx->comm);
  ctx->comm = ctx->comm_side = nullptr;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  NcclComm* c = new (std::nothrow) NcclComm();
  NcclComm* cs = new (std::nothrow) NcclComm();
  if (!c || !cs) {
    delete c;
    delete cs;
    return RANDUTV_ERR_ALLOC;
  }
  c->api = cs->api = api;
  c->rank = cs->rank = rank;
  c->nranks = cs->nranks = nranks;
  ncclResult_t r = api->CommInitRank(&c->comm, nranks, id, rank);
  if (r == ncclSuccess) r = api->CommSplit(c->comm, 0, rank, &cs->comm, nullptr);
  if (r != ncclSuccess) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "ncclCommInitRank/Split: %s", api->GetErrorString(r));
    set_last_error(g_nccl_err, cudaErrorUnknown);
    delete cs;
    delete c;
    return RANDUTV_ERR_NCCL;
  }
  c->partner = cs;
  cs->partner = c;
  ctx->comm = c;
  ctx->comm_side = cs;
  return 0;
}

RANDUTV_API int randutv_factor_dist(randutv_ctx* ctx, int64_t m, int64_t n, double* A_local, int64_t lda,
                                    int64_t b, int q, uint64_t seed, unsigned flags, double* U_local, int64_t ldu,
                                    double* V_local, int64_t ldv) {
  RUTV_TRY(begin_call(ctx));
  if (!ctx->comm) return RANDUTV_ERR_NOCOMM;
  return dist_factor(ctx, ctx->comm, ctx->comm_side, m, n, A_local, lda, b, q, seed, flags, U_local, ldu, V_local,
                     ldv, 0, nullptr);
}

RANDUTV_API int randutv_factor_dist_rank(randutv_ctx* ctx, int64_t m, int64_t n, double* A_local, int64_t lda,
                                         int64_t k, int64_t b, int q, uint64_t seed, unsigned flags, double* Uk_local,
                                         int64_t ldu, double* V_local, int64_t ldv, double* resid_fro) {
  RUTV_TRY(begin_call(ctx));
  if (!ctx->comm) return RANDUTV_ERR_NOCOMM;
  if (k < 1) return -14;
  return dist_factor(ctx, ctx->comm, ctx->comm_side, m, n, A_local, lda, b, q, seed, flags, Uk_local, ldu, V_local,
                     ldv, k, resid_fro);
}

RANDUTV_API int randutv_factor_dist_host_loopback(int device, int nranks, int64_t m, int64_t n,
                                                  double* const* A_locals_host, int64_t lda, int64_t b, int q,
                                                  uint64_t seed, unsigned flags, size_t device_cache_bytes,
                                                  double* const* U_locals_host, int64_t ldu,
                                                  double* const* V_locals_host, int64_t ldv) {
  if (nranks < 1 || nranks > kMaxLoopRanks) return -2;
  if (!A_locals_host) return -5;
  const bool uv = !(flags & RANDUTV_NO_UV);
  if (uv && (!U_locals_host || !V_locals_host)) return -12;
  LoopShared sh(nranks);
  std::vector<int> status(nranks, 0);
  std::vector<std::thread> th;
  std::vector<LoopComm*> comms(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    comms[r] = new LoopComm();
    comms[r]->sh = &sh;
    comms[r]->rank = r;
    comms[r]->nranks = nranks;
  }
  for (int r = 0; r < nranks; ++r) {
    th.emplace_back([&, r] {
      int st = 0;
      randutv_ctx* ctx = nullptr;
      cudaStream_t s = nullptr;
      if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
        st = RANDUTV_ERR_CUDA;
      if (st == 0) st = randutv_create(&ctx, device, s);
      if (st == 0) {
        comms[r]->sms = ctx->sms;
        st = dist_host_factor(ctx, comms[r], m, n, A_locals_host[r], lda, b, q, seed, flags, device_cache_bytes,
                              uv ? U_locals_host[r] : nullptr, ldu, uv ? V_locals_host[r] : nullptr, ldv, nullptr);
      }
      if (ctx) randutv_destroy(ctx);
      if (s) cudaStreamDestroy(s);
      status[r] = st;
    });
  }
  for (auto& t : th) t.join();
  for (LoopComm* c : comms) delete c;
  for (int r = 0; r < nranks; ++r)
    if (status[r] != 0) return status[r];
  return 0;
}

RANDUTV_API int randutv_factor_dist_loopback(int device, int nranks, int64_t m, int64_t n, double* const* A_locals,
                                             int64_t lda, int64_t b, int q, uint64_t seed, unsigned flags,
                                             double* const* U_locals, int64_t ldu, double* const* V_locals,
                                             int64_t ldv, int64_t k, double* resid_fro) {
  if (k < 0) return -15;
  if (k > 0 && !resid_fro) return -16;
  if (nranks < 1 || nranks > kMaxLoopRanks) return -2;
  if (!A_locals) return -5;
  const bool uv = !(flags & RANDUTV_NO_UV);
  if (uv && (!U_locals || !V_locals)) return -11;
  LoopShared sh(nranks);
  std::vector<int> status(nranks, 0);
  std::vector<std::thread> th;
  std::vector<LoopComm*> comms(2 * nranks, nullptr);
  for (int r = 0; r < 2 * nranks; ++r) {
    comms[r] = new LoopComm();
    comms[r]->sh = &sh;  // main and side collectives share the barrier: issued in program order
    comms[r]->rank = r % nranks;
    comms[r]->nranks = nranks;
  }
  for (int r = 0; r < nranks; ++r) {
    th.emplace_back([&, r] {
      int st = 0;
      randutv_ctx* ctx = nullptr;
      cudaStream_t s = nullptr;
      if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        st = RANDUTV_ERR_CUDA;
      }
      if (st == 0) st = randutv_create(&ctx, device, s);
      if (st == 0) st = begin_call(ctx);
      if (st == 0) {
        comms[r]->sms = comms[nranks + r]->sms = ctx->sms;
        double rho = 0.0;
        st = dist_factor(ctx, comms[r], comms[nranks + r], m, n, A_locals[r], lda, b, q, seed, flags,
                         uv ? U_locals[r] : nullptr, ldu, uv ? V_locals[r] : nullptr, ldv, k, k > 0 ? &rho : nullptr);
        if (st == 0 && k > 0 && r == 0) *resid_fro = rho;
      }
      if (ctx) randutv_destroy(ctx);
      if (s) cudaStreamDestroy(s);
      status[r] = st;
    });
  }
  for (auto& t : th) t.join();
  for (LoopComm* c : comms) delete c;
  for (int r = 0; r < nranks; ++r)
    if (status[r] != 0) return status[r];
  return 0;
}

}  // extern "C"
