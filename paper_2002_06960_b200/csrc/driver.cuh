// Host-driver internals shared by the single-GPU driver (randutv.cu) and the
// column-sharded multi-GPU driver (dist.cu): the context, the workspace
// carving and the compact-WY application helpers.  Not part of the C ABI.
#pragma once
#include "common.cuh"

#include <algorithm>

namespace rutv {

// 1-D block-cyclic column layout of the sharded paths (dist.cu, host.cu)
struct Layout {
  i64 m, n, b;
  int P, p;
  i64 nblocks;
  i64 width(i64 j) const { return std::min(b, n - j * b); }
  // local column count of rank q
  i64 ncols(int q) const {
    i64 c = 0;
    for (i64 j = q; j < nblocks; j += P) c += width(j);
    return c;
  }
  // number of rank q's blocks with global index < i
  i64 lb_before(int q, i64 i) const { return i > q ? (i - q + P - 1) / P : 0; }
  // local column offset of rank q's first block with global index >= i
  i64 lcol(int q, i64 i) const { return lb_before(q, i) * b; }
  i64 trailing_cols(int q, i64 i) const { return ncols(q) - lcol(q, i); }
  i64 max_trailing(i64 i) const {
    i64 mx = 0;
    for (int q = 0; q < P; ++q) mx = std::max(mx, trailing_cols(q, i));
    return mx;
  }
  static i64 row0(i64 rows, int P, int q) { return rows * q / P; }
};

// Collectives of the sharded paths: NCCL or the single-GPU loopback (dist.cu)
struct Comm {
  int rank = 0, nranks = 1;
  int* dflag = nullptr;  // one device int for the pre-collective agreement (agree())
  virtual ~Comm() {
    if (dflag) cudaFree(dflag);
  }
  // wait for stream `s`, whose work includes this communicator's collectives:
  // NCCL polls the communicator's asynchronous error state and aborts it on
  // an error or after the timeout instead of blocking forever on a dead peer
  virtual int sync(cudaStream_t s) {
    RUTV_CUDA(cudaStreamSynchronize(s));
    return 0;
  }
  virtual int allreduce_sum(double* buf, i64 count, cudaStream_t s) = 0;
  // recv holds nranks * count doubles, rank q's block at q * count
  virtual int allgather(const double* send, double* recv, i64 count, cudaStream_t s) = 0;
  virtual int bcast(double* buf, i64 count, int root, cudaStream_t s) = 0;
  virtual int allreduce_min_int(int* buf, i64 count, cudaStream_t s) = 0;
  // row chunks of a pipelined GEMM -> AllReduce (1: no pipelining; the
  // loopback's collectives synchronise the host, so chunking only adds barriers)
  virtual int chunks() const { return 1; }
  // collectives can be captured into a CUDA graph (NCCL: yes; loopback: no)
  virtual bool capturable() const { return false; }
};


}  // namespace rutv

struct randutv_ctx {
  int magic;
  int device;
  cudaStream_t stream;
  int sms;
  void* ws;
  size_t ws_bytes;
  // ws was used by a RANDUTV_ASYNC call (maybe captured into a graph): a
  // growth retires it to `retired` (freed by randutv_destroy) instead of
  // freeing it under the graph
  bool ws_captured;
  std::vector<void*> retired;
  randutv_stats stats;
  // host-staging buffers of the literal (host pointer) entry
  double* stage;
  size_t stage_bytes;
  rutv::Profiler prof;
  // side stream (high priority) for the small SVD + folds, and its two events
  cudaStream_t side;
  cudaEvent_t eR, eF;
  // V stream: the V update (S5 on V) of a step runs concurrently with the QR of
  // the column block and the T updates (eWv: W_V ready; eV: V update done)
  cudaStream_t vstr;
  cudaEvent_t eWv, eV;
  // U update of step i on the V stream (eWu: W_U ready; eU: U update done)
  cudaEvent_t eWu, eU;
  // eS: a step reached its QR(Y) (the deferred U update starts); eFuv: the
  // side stream's U / V folds done
  cudaEvent_t eS, eFuv, eUf;  // eUf: a deferred U fold read U_s
  cudaEvent_t eUb[2];         // the deferred U update reading (W_U, T_U) buffer j done
  // multi-GPU communicators (randutv_comm_init): main-stream and side-stream
  rutv::Comm* comm;
  rutv::Comm* comm_side;
  // copy stream of the literal host-pointer entry (column blocks drain to the
  // host while the factorisation runs)
  cudaStream_t cps;
  // device status word of the last RANDUTV_ASYNC call (randutv_wait)
  int* async_status;
  // the last RANDUTV_ASYNC call was sharded: randutv_wait waits through the
  // communicator (asynchronous-error polling, timeout)
  bool async_dist;
  // sharded path: the stream its main-stream collectives run on (chunked
  // AllReduces overlap the GEMMs producing the next chunk)
  cudaStream_t cstr;
  cudaEvent_t ecomm[8];
  // GEMM tile-scheduler counters: [0..1] main stream, [2..3] side stream (zeroed once)
  int* sched;
  int jacobi_max_sweeps;  // 0 = the default 30 (randutv_set_option)
  int64_t oversample;     // p extra sample columns (randutv_set_option, reading A28)
  rutv::Launch with_opts(rutv::Launch l) const {
    if (jacobi_max_sweeps > 0) l.jacobi_max_sweeps = jacobi_max_sweeps;
    return l;
  }
  rutv::Launch launch() { return with_opts(rutv::Launch{stream, &stats.kernel_launches, sms, &prof, sched}); }
  rutv::Launch v_launch() {
    rutv::Launch l{vstr, &stats.kernel_launches, sms, &prof, nullptr};
    l.oneshot = true;
    return with_opts(l);
  }
  rutv::Launch side_launch() {
    return with_opts(rutv::Launch{side, &stats.kernel_launches, sms, &prof, sched ? sched + 2 : nullptr});
  }
};

namespace rutv {

constexpr int kMagic = 0x52555456;  // "RUTV"
constexpr i64 kAlign = 256;

struct Carver {
  char* base;
  size_t off;
  size_t cap;
  bool dry;
  template <typename Tp>
  Tp* take(i64 elems) {
    size_t bytes = ((size_t)(elems > 0 ? elems : 1) * sizeof(Tp) + kAlign - 1) / kAlign * kAlign;
    Tp* p = dry ? nullptr : reinterpret_cast<Tp*>(base + off);
    off += bytes;
    return p;
  }
};

// All per-call device buffers.
struct Work {
  double *G, *Y, *Z, *Z2, *Wv, *Wu, *TV, *TU, *tauV, *tauU;
  double *Us, *Vs, *d;
  double *jac, *gemm_ws, *red, *scal;
  i64 jac_elems, gemm_ws_elems;
  int *status, *flag;
  QrWork qw;
  double* lefts;  // truncated-U records
  i64 lefts_elems;
  double* Twork;  // m x n working T for the truncated variant
  double* Zf;     // fold temporaries of the side stream (max(m,n) x b)
  double* Acat;   // fused S5/S7 update operands: [Z2(k:m) | W_U]  (m x 2b)
  double* Bt;     //                              [W2 | Y^T]       (n x 2b)
  double *Zv, *Zv2, *gemm_ws_v;  // temporaries of the V stream (n x b each; split-K)
  double *Wu2, *TU2;             // second (W_U, T_U) buffer (deferred U update)
  double *osR, *osU, *osV, *osd, *osjac;  // oversampling: Rayleigh-Ritz SVD (b x b each; b = b + p)
};

i64 gemm_ws_elems_for(i64 m, i64 n, i64 b);
size_t carve(Carver& c, Work& w, i64 m, i64 n, i64 b, i64 lefts_K, bool twork);
int ensure_ws(randutv_ctx* ctx, size_t bytes);
int prepare(randutv_ctx* ctx, Work& w, i64 m, i64 n, i64 b, i64 lefts_K, bool twork);
int begin_call(randutv_ctx* ctx);
// synchronise the ctx stream and turn the device status word into the return code
int finish(randutv_ctx* ctx, const Work& w);
i64 sampled_steps(i64 n, i64 b);
// dist.cu: release a communicator (NULL is a no-op)
void comm_free(Comm* c);
// host.cu: the sharded host-streamed factorisation on one rank (NEXT-1)
int dist_host_factor(randutv_ctx* ctx, Comm* comm, int64_t m, int64_t n, double* A_local, int64_t lda, int64_t b, int q,
                     uint64_t seed, unsigned flags, size_t cache_bytes, double* U_local, int64_t ldu,
                     double* V_local, int64_t ldv, randutv_host_report* report);
// dist.cu: the layout kernels (global trailing order <-> a rank's local order)
int launch_cyclic_gather_rows(const Launch& L, i64 s, i64 cols, i64 k, i64 b, int P, i64 i, const double* Yall,
                              i64 ldc, i64 stride, double* Y, i64 ldy);
int launch_cyclic_scatter_rows(const Launch& L, i64 sl, i64 cols, i64 k, i64 b, int P, int p, i64 lb0,
                               const double* W, i64 ldw, double* Wl, i64 ldl);
// dist.cu: wait for a stream whose work includes the communicator's collectives
int comm_sync(Comm* c, cudaStream_t s);
int start_status(randutv_ctx* ctx, const Work& w);
int check_finite(randutv_ctx* ctx, const Launch& L, const Work& w, i64 m, i64 n, const double* A, i64 lda);

// X(rows x s, ldx) -= ((X W) Tf) W^T : the right application of Q = I - W Tf W^T
int apply_right(const Launch& L, Work& w, i64 rows, i64 s, i64 bw, double* X, i64 ldx, const double* W, i64 ldw,
                const double* Tf, i64 ldtf);
// X(r x c) -= W Tf^T (W^T X): the left application of Q^T
int apply_left_t(const Launch& L, Work& w, i64 r, i64 c, i64 bw, double* X, i64 ldx, const double* W, i64 ldw,
                 const double* Tf, i64 ldtf);
// S5 + S7 of the columns right of block i as one rank-2b update (randutv.cu)
int fused_right_left(const Launch& L, Work& w, i64 m, i64 r, i64 b, i64 kk, i64 c, double* X, i64 ldx,
                     const double* W2, i64 ldw2, const double* Z2, i64 ldz, const double* Wu, i64 ldwu,
                     const double* TU, i64 ldtu, i64 top = -1);
bool fuse_left();
// X(rows x bw) := X M  (M bw x bw), via the temporary Zt
int right_mult_inplace(const Launch& L, double* Zt, i64 rows, i64 bw, double* X, i64 ldx, const double* M, i64 ldm);
// X(bw x cols) := M^T X
int left_mult_t_inplace(const Launch& L, double* Zt, i64 bw, i64 cols, double* X, i64 ldx, const double* M, i64 ldm);

}  // namespace rutv
