// Host-streamed randUTV: A, U and V stay in (pinned)
// host memory and stream through a bounded device panel cache -- the GPU
// analogue of the paper's out-of-core setting, where the matrix lives on disk
// and blocks move through an LRU cache in RAM ("cache"
// dispatcher) while a dedicated I/O thread overlaps the transfers with the
// computation ("cache + overlap").
//
// Unit of transfer: a column panel (all rows x b columns) of T (= A, updated
// in place), U or V.  The cache holds C panel slots (device_cache_bytes /
// (max(m,n) b 8 bytes), at least 3); victims are least recently used, dirty
// victims are written back first.  Every pass over the trailing panels runs
// in the direction opposite to the previous pass ("serpentine"), so an LRU
// cache smaller than the pass keeps the panels the next pass starts with
// (cyclic sweeps larger than an LRU cache never hit).
// Copies run on two copy streams (H2D prefetch of the next panel of the pass,
// D2H write-back of victims) and overlap the DMMA work on the compute stream;
// events order slot reuse.  Per sampled step i (k = i b), panels j >= i,
// 2q + 2 passes over T (step 0: one more, its S2 pass):
//   2q passes (R)  Z = sum_j T_j(k:m) Y_j ; Y_j = T_j(k:m)^T Z           S3
//                  (rows k:m only: a panel fetched here loads rows k:m;
//                  rows 0:k follow when a later pass needs them)
//   QR(Y) on the device                                                  S4
//   pass     (R)   Z = sum_j T_j W_j (all m rows)                        S5
//   panel i        S5 update, QR of rows k:m (S6), Jacobi SVD of the
//                  diagonal block, T11 = diag d, A01 V_s                 S5, S6, S8, S9
//   pass     (RW)  panels j > i: S5 update, S7 left update, U_s^T fold of
//                  rows k:k+b, and the NEXT step's sample
//                  Y'_j = T_j(k+b:m)^T G'  while the panel is resident   S5, S7, S9, S1+S2
//   V, U           read pass (X W) + RW pass (X -= ...) over their trailing
//                  panels, then U_i U_s, V_i V_s                          S5, S7, S9
// The arithmetic is that of the in-HBM driver (same kernels, same reflector
// conventions); only sums over panels are split (GEMM accumulation with
// beta = 1), so results agree with randutv_factor_ex to rounding.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "driver.cuh"

namespace rutv {

namespace {

struct HostMat {
  double* h;
  i64 rows, cols, ld;
  i64 npanels;
};

struct Slot {
  double* d = nullptr;
  int mat = -1;
  i64 panel = -1;
  i64 lo = 0;  // rows [lo, rows) of the panel are resident (sample passes need only k..m)
  bool dirty = false;
  int pins = 0;
  uint64_t last = 0;
  int64_t next_use = 0;  // Belady: position of the panel's next access in the plan
  cudaEvent_t ready = nullptr, idle = nullptr, clean = nullptr;
};

struct CopyTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<size_t, size_t>> h2d, d2h;
  int mark(cudaStream_t s, size_t* idx) {
    if (used == pool.size()) {
      cudaEvent_t e;
      RUTV_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    RUTV_CUDA(cudaEventRecord(pool[used], s));
    *idx = used++;
    return 0;
  }
  ~CopyTimer() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

struct PanelCache {
  std::vector<HostMat> mats;
  std::vector<std::vector<int>> where;  // mat -> panel -> slot (-1: host only)
  // mat -> panel -> event after the panel's latest write-back (a re-fetch of the
  // panel must not read host memory before its write-back has landed)
  std::vector<std::vector<cudaEvent_t>> wbev;
  std::vector<Slot> slots;
  double* base = nullptr;
  i64 slot_elems = 0, b = 0;
  cudaStream_t comp = nullptr, h2d = nullptr, d2h = nullptr;
  cudaEvent_t h2d_done = nullptr;
  uint64_t clock = 0;
  randutv_host_report* rep = nullptr;
  CopyTimer timer;
  // Belady eviction (T-only runs): the driver's panel access sequence of T is
  // known in advance (build_plan); every get() of T is matched against it and
  // the victim is the unpinned slot whose next use lies farthest ahead.  A
  // mismatch (an access the plan does not predict) falls back to LRU.
  int plan_mat = -1;
  std::vector<i64> plan, nxt;  // plan[t]: panel of access t; nxt[t]: next access of that panel (or INT64_MAX)
  i64 cursor = 0;
  bool use_plan = false;
  int add_mat(double* h, i64 rows, i64 cols, i64 ld) {
    mats.push_back(HostMat{h, rows, cols, ld, (cols + b - 1) / b});
    where.emplace_back((size_t)mats.back().npanels, -1);
    wbev.emplace_back((size_t)mats.back().npanels, nullptr);
    return (int)mats.size() - 1;
  }
  i64 width(int mat, i64 p) const { return std::min(b, mats[mat].cols - p * b); }

  int init(i64 nslots, double* dbase) {
    base = dbase;
    slots.resize((size_t)nslots);
    for (i64 s = 0; s < nslots; ++s) {
      slots[s].d = base + s * slot_elems;
      RUTV_CUDA(cudaEventCreateWithFlags(&slots[s].ready, cudaEventDisableTiming));
      RUTV_CUDA(cudaEventCreateWithFlags(&slots[s].idle, cudaEventDisableTiming));
      RUTV_CUDA(cudaEventCreateWithFlags(&slots[s].clean, cudaEventDisableTiming));
    }
    return 0;
  }
  void destroy() {
    for (auto& v : wbev)
      for (cudaEvent_t e : v)
        if (e) cudaEventDestroy(e);
    wbev.clear();
    for (Slot& s : slots) {
      if (s.ready) cudaEventDestroy(s.ready);
      if (s.idle) cudaEventDestroy(s.idle);
      if (s.clean) cudaEventDestroy(s.clean);
    }
    slots.clear();
  }

  int write_back(Slot& s) {
    if (!s.dirty) return 0;
    const HostMat& M = mats[s.mat];
    const i64 w = width(s.mat, s.panel);
    RUTV_CUDA(cudaStreamWaitEvent(d2h, s.idle, 0));
    size_t e0 = 0, e1 = 0;
    if (timer.on) RUTV_TRY(timer.mark(d2h, &e0));
    RUTV_CUDA(cudaMemcpy2DAsync(M.h + s.panel * b * M.ld + s.lo, M.ld * 8, s.d + s.lo, M.rows * 8,
                                (M.rows - s.lo) * 8, w, cudaMemcpyDeviceToHost, d2h));
    if (timer.on) {
      RUTV_TRY(timer.mark(d2h, &e1));
      timer.d2h.push_back({e0, e1});
    }
    RUTV_CUDA(cudaEventRecord(s.clean, d2h));
    cudaEvent_t& we = wbev[s.mat][s.panel];
    if (!we) RUTV_CUDA(cudaEventCreateWithFlags(&we, cudaEventDisableTiming));
    RUTV_CUDA(cudaEventRecord(we, d2h));
    rep->d2h_bytes += (M.rows - s.lo) * w * 8;
    s.dirty = false;
    return 0;
  }

  int victim(int* out) {
    int best = -1;
    for (int s = 0; s < (int)slots.size(); ++s) {
      if (slots[s].pins > 0) continue;
      if (slots[s].mat < 0) {
        best = s;
        break;
      }
      if (best < 0) {
        best = s;
      } else if (use_plan) {
        if (slots[s].next_use > slots[best].next_use) best = s;
      } else if (slots[s].last < slots[best].last) {
        best = s;
      }
    }
    if (best < 0) return RANDUTV_ERR_ALLOC;  // every slot pinned: cannot happen with >= 3 slots
    *out = best;
    return 0;
  }

  // H2D of rows [lo, hi) of (mat, panel) into slot v (after its earlier users)
  int load_rows(Slot& v, int mat, i64 panel, i64 lo, i64 hi) {
    const HostMat& M = mats[mat];
    const i64 w = width(mat, panel);
    if (wbev[mat][panel]) RUTV_CUDA(cudaStreamWaitEvent(h2d, wbev[mat][panel], 0));
    size_t e0 = 0, e1 = 0;
    if (timer.on) RUTV_TRY(timer.mark(h2d, &e0));
    RUTV_CUDA(cudaMemcpy2DAsync(v.d + lo, M.rows * 8, M.h + panel * b * M.ld + lo, M.ld * 8, (hi - lo) * 8, w,
                                cudaMemcpyHostToDevice, h2d));
    if (timer.on) {
      RUTV_TRY(timer.mark(h2d, &e1));
      timer.h2d.push_back({e0, e1});
    }
    rep->h2d_bytes += (hi - lo) * w * 8;
    return 0;
  }

  // make rows [lo, rows) of (mat, panel) resident; `load` = false gives an
  // uninitialised slot (the caller overwrites the whole panel, e.g. U := I)
  int fetch(int mat, i64 panel, bool load, int* out, i64 lo = 0) {
    const HostMat& M = mats[mat];
    int s = where[mat][panel];
    if (s >= 0) {
      Slot& v = slots[s];
      if (load && lo < v.lo) {  // resident, but the rows above are needed now
        RUTV_CUDA(cudaStreamWaitEvent(h2d, v.idle, 0));
        RUTV_TRY(load_rows(v, mat, panel, lo, v.lo));
        v.lo = lo;
        RUTV_CUDA(cudaEventRecord(v.ready, h2d));
      }
      ++rep->cache_hits;
      *out = s;
      return 0;
    }
    ++rep->cache_misses;
    RUTV_TRY(victim(&s));
    Slot& v = slots[s];
    if (v.mat >= 0) {
      RUTV_TRY(write_back(v));
      where[v.mat][v.panel] = -1;
    }
    v.mat = mat;
    v.panel = panel;
    v.dirty = false;
    v.last = ++clock;
    v.lo = load ? lo : 0;
    where[mat][panel] = s;
    RUTV_CUDA(cudaStreamWaitEvent(h2d, v.idle, 0));
    RUTV_CUDA(cudaStreamWaitEvent(h2d, v.clean, 0));
    if (load) RUTV_TRY(load_rows(v, mat, panel, lo, M.rows));
    RUTV_CUDA(cudaEventRecord(v.ready, h2d));
    *out = s;
    return 0;
  }

  // pin (mat, panel) for compute on `comp`; returns the device panel (ld = rows)
  int get(int mat, i64 panel, double** d, bool load = true, i64 lo = 0) {
    int64_t nu = 0;
    if (use_plan && mat == plan_mat) {
      if (cursor < (i64)plan.size() && plan[cursor] == panel) {
        nu = nxt[cursor++];
      } else {
        use_plan = false;  // the run left the plan: LRU from here on
      }
    }
    int s;
    RUTV_TRY(fetch(mat, panel, load, &s, lo));
    Slot& v = slots[s];
    v.pins++;
    v.last = ++clock;
    v.next_use = nu;
    RUTV_CUDA(cudaStreamWaitEvent(comp, v.ready, 0));
    *d = v.d;
    return 0;
  }
  int put(int mat, i64 panel, bool dirty) {
    Slot& v = slots[where[mat][panel]];
    v.pins--;
    v.dirty = v.dirty || dirty;
    RUTV_CUDA(cudaEventRecord(v.idle, comp));
    return 0;
  }
  // `ahead` = how many accesses of the plan lie before this panel's use
  int prefetch(int mat, i64 panel, i64 lo = 0, i64 ahead = 0) {
    if (panel < 0 || panel >= mats[mat].npanels) return 0;
    int s;
    RUTV_TRY(fetch(mat, panel, true, &s, lo));
    // the prefetched panel is (one of) the plan's next accesses: not a victim before its use
    if (use_plan && mat == plan_mat) slots[s].next_use = cursor + ahead;
    return 0;
  }
  int flush() {
    for (Slot& s : slots)
      if (s.mat >= 0) RUTV_TRY(write_back(s));
    return 0;
  }
};

// The panel accesses of T the driver makes, in order (host_sampled_step /
// host_final_step; pass directions as pass() with R.dir = (i & 1) == 0 at each
// step): [step_begin only: the S2 pass over panels i..], 2q power passes, the
// T W_V read pass, panel i, the read-write pass over panels i+1..; the final
// block.  paper_2002_06960_b200/flops.py host_stream_traffic replays the same
// sequence (the PCIe-byte model).
void build_plan(i64 n, i64 b, int q, i64 nsamp, i64 step_begin, i64 step_end, std::vector<i64>& plan,
                std::vector<i64>& nxt) {
  const i64 np = (n + b - 1) / b;
  plan.clear();
  const i64 last = std::min(step_end, nsamp);
  for (i64 i = step_begin; i < last; ++i) {
    bool fwd = (i & 1) == 0;
    auto pass = [&](i64 p0) {
      for (i64 t = 0; t < np - p0; ++t) plan.push_back(fwd ? p0 + t : np - 1 - t);
      fwd = !fwd;
    };
    if (i == step_begin) pass(i);  // S2 (the previous step's fused pass took it otherwise)
    for (int qq = 0; qq < 2 * q; ++qq) pass(i);
    pass(i);                // T W_V
    plan.push_back(i);      // panel i
    pass(i + 1);            // S5 + S7 + fold + next S2
  }
  if (step_end > nsamp) plan.push_back(nsamp);
  nxt.assign(plan.size(), INT64_MAX);
  std::vector<i64> seen((size_t)np, INT64_MAX);
  for (i64 t = (i64)plan.size() - 1; t >= 0; --t) {
    nxt[t] = seen[plan[t]];
    seen[plan[t]] = t;
  }
}

// RUTV_HOST_EVICT=lru disables the Belady plan (comparison only)
bool belady_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_HOST_EVICT");
    v = (e && strcmp(e, "lru") == 0) ? 0 : 1;
  }
  return v != 0;
}

struct HostRun {
  randutv_ctx* ctx;
  Launch L;
  Work w;
  PanelCache pc;
  int mT = -1, mU = -1, mV = -1;
  i64 m, n, b;
  int q;
  uint64_t seed;
  bool dir = false;        // direction of the next pass (serpentine)
  bool y_ready = false;    // Y of the next step was taken by the previous step's fused pass
  // Deferred U / V accumulation: up to G steps' (W, T, S) of one matrix are
  // merged into ONE compact-WY transform and applied in one read + one RW pass
  // (see flush_uv).  G <= 1: per-step application.
  struct Batch {
    int mat = -1;
    i64 rows = 0;             // U: m, V: n (the matrix's column-index space)
    double* W = nullptr;      // rows x G b: block l = [0 (rows < k_l); W_l]
    double* T = nullptr;      // G blocks of b x b: T_l
    double* S = nullptr;      // G blocks of b x b: the S9 fold factor (U_s or V_s)
    double* Tc = nullptr;     // G b x G b: the merged T
    std::vector<i64> k;       // first column of each pending step
  };
  int G = 1;
  Batch bu, bv;
  double *Zb = nullptr, *Zb2 = nullptr;  // max(m, n) x G b temporaries of the merged apply
  // sharded (randutv_factor_dist_host): the rank's communicator and layout;
  // Yl / Wl = the rank's rows of Y / W_V (maxs x b), Yall the all-gathered
  // chunks, wbuf = the owner's broadcast [W_U | T_U | U_s | V_s]
  Comm* comm = nullptr;
  Layout lay{};
  double *Yl = nullptr, *Yall = nullptr, *Wl = nullptr, *wbuf = nullptr;
  i64 maxs = 0;
};

// Visit panels [p0, p1) of `mat` in the current serpentine direction with a
// one-panel prefetch; f(panel, device ptr) enqueues the work on the compute stream.
// RUTV_HOST_PREFETCH: panels of a pass fetched ahead of the one computed (default 2)
i64 prefetch_depth() {
  static i64 v = -1;
  if (v < 0) {
    const char* e = getenv("RUTV_HOST_PREFETCH");
    v = e ? atoll(e) : 2;
    if (v < 1) v = 1;
  }
  return v;
}

template <class F>
int pass(HostRun& R, int mat, i64 p0, i64 p1, bool dirty, F&& f, i64 lo = 0) {
  const bool fwd = R.dir;
  R.dir = !R.dir;
  const i64 cnt = p1 - p0;
  // never prefetch more than the cache can hold next to the pinned panel
  const i64 depth = std::min<i64>(prefetch_depth(), (i64)R.pc.slots.size() - 2);
  for (i64 t = 0; t < cnt; ++t) {
    const i64 j = fwd ? p0 + t : p1 - 1 - t;
    double* d;
    RUTV_TRY(R.pc.get(mat, j, &d, true, lo));
    for (i64 a = 1; a <= depth && t + a < cnt; ++a)
      RUTV_TRY(R.pc.prefetch(mat, fwd ? j + a : j - a, lo, a - 1));
    RUTV_TRY(f(j, d));
    RUTV_TRY(R.pc.put(mat, j, dirty));
  }
  return 0;
}

// right update of the trailing panels [p0, np) of matrix `mat` (rows x *):
// X -= ((X W) Tf) W^T with W (ld ldw) rows aligned to panel p0's first column
int stream_apply_right(HostRun& R, int mat, i64 p0, i64 bw, const double* W, i64 ldw, const double* Tf, i64 ldtf,
                       double* Z = nullptr, double* Z2 = nullptr) {
  const HostMat& M = R.pc.mats[mat];
  const i64 rows = M.rows;
  Work w = R.w;
  if (Z) {
    w.Z = Z;
    w.Z2 = Z2;
  }
  // Z = sum_j X_j W_j   (fixed panel order inside a pass is not needed for
  // correctness; the GEMM accumulation is beta = 1)
  RUTV_TRY(launch_fill(R.L, rows, bw, 0.0, w.Z, rows));
  RUTV_TRY(pass(R, mat, p0, M.npanels, false, [&](i64 j, double* X) {
    const i64 wj = R.pc.width(mat, j);
    return launch_dgemm(R.L, false, false, rows, bw, wj, 1.0, X, rows, W + (j - p0) * R.b, ldw, 1.0, w.Z, rows,
                        nullptr, 0);
  }));
  RUTV_TRY(launch_dgemm(R.L, false, false, rows, bw, bw, 1.0, w.Z, rows, Tf, ldtf, 0.0, w.Z2, rows, nullptr, 0));
  return pass(R, mat, p0, M.npanels, true, [&](i64 j, double* X) {
    const i64 wj = R.pc.width(mat, j);
    return launch_dgemm(R.L, false, true, rows, wj, bw, -1.0, w.Z2, rows, W + (j - p0) * R.b, ldw, 1.0, X, rows,
                        nullptr, 0);
  });
}

// S8 + the T part of S9 on panel i (width bw): T11 := diag(d), T(0:k, blk) := T(0:k, blk) V_s.
// U_s^T T(k:k+b, k+b:n) is folded by the caller's pass over the trailing panels.
int host_svd_T(HostRun& R, i64 i, i64 bw, double* X) {
  Work& w = R.w;
  const i64 k = i * R.b;
  double* T11 = X + k;
  RUTV_TRY(launch_jacobi_svd(R.L, bw, T11, R.m, w.Us, w.d, w.Vs, w.status, (int)(i + 1), w.jac, w.jac_elems));
  RUTV_TRY(launch_set_diag(R.L, bw, w.d, T11, R.m));
  return right_mult_inplace(R.L, w.Zf, k, bw, X, R.m, w.Vs, bw);  // A01 V_s
}

// the U and V parts of S9: U(:, blk) := U(:, blk) U_s, V(:, blk) := V(:, blk) V_s
int host_fold_uv(HostRun& R, i64 i, i64 bw) {
  Work& w = R.w;
  double* X;
  // (panel rows: all of U / V on one GPU, the rank's row range when sharded)
  if (R.mU >= 0) {
    const i64 rows = R.pc.mats[R.mU].rows;
    RUTV_TRY(R.pc.get(R.mU, i, &X));
    RUTV_TRY(right_mult_inplace(R.L, w.Zf, rows, bw, X, rows, w.Us, bw));
    RUTV_TRY(R.pc.put(R.mU, i, true));
  }
  if (R.mV >= 0) {
    const i64 rows = R.pc.mats[R.mV].rows;
    RUTV_TRY(R.pc.get(R.mV, i, &X));
    RUTV_TRY(right_mult_inplace(R.L, w.Zf, rows, bw, X, rows, w.Vs, bw));
    RUTV_TRY(R.pc.put(R.mV, i, true));
  }
  return 0;
}

// Deferred U / V updates.  Step l of a batch applies X := X H_l D_l with
// H_l = I - W_l T_l W_l^T (columns k_l:) and D_l = diag(I, S_l, I) (the S9
// fold of block l).  Since H D = D (D^T H D) and every D_j acts on its own
// column block, the batch equals X D_0 ... D_{L-1} (I - W^f T_c W^f^T) with
// W^f = D^T [W_0 .. W_{L-1}] (block row j of W multiplied by S_j^T) and T_c
// the merged forward T (T_c(0:lb, lb:(l+1)b) = -T_c(0:lb, 0:lb) W^f_{0:l}^T W^f_l T_l).
int flush_uv(HostRun& R, HostRun::Batch& B) {
  const i64 L = (i64)B.k.size();
  if (L == 0) return 0;
  Work& w = R.w;
  const i64 b = R.b, k0 = B.k[0], rows = B.rows, ldc = R.G * b, h = rows - k0;
  double* Wf = B.W + k0;  // rows k0:rows of the batch's W, ld rows
  // D: the folds of the L blocks
  const i64 prow = R.pc.mats[B.mat].rows;  // panel rows (the rank's row range when sharded)
  for (i64 l = 0; l < L; ++l) {
    double* X;
    RUTV_TRY(R.pc.get(B.mat, B.k[l] / b, &X));
    RUTV_TRY(right_mult_inplace(R.L, w.Zf, prow, b, X, prow, B.S + l * b * b, b));
    RUTV_TRY(R.pc.put(B.mat, B.k[l] / b, true));
  }
  // W^f = D^T W: block row j (rows k_j:k_j+b) of the blocks l <= j
  for (i64 j = 0; j < L; ++j)
    RUTV_TRY(left_mult_t_inplace(R.L, w.Zf, b, (j + 1) * b, B.W + B.k[j], rows, B.S + j * b * b, b));
  // T_c
  RUTV_TRY(launch_fill(R.L, L * b, L * b, 0.0, B.Tc, ldc));
  for (i64 l = 0; l < L; ++l) {
    RUTV_TRY(launch_copy(R.L, b, b, B.T + l * b * b, b, B.Tc + l * b * (ldc + 1), ldc));
    if (l == 0) continue;
    const i64 lb = l * b;
    RUTV_TRY(launch_dgemm(R.L, true, false, lb, b, h, 1.0, Wf, rows, Wf + lb * rows, rows, 0.0, w.Z, lb, w.gemm_ws,
                          w.gemm_ws_elems));
    RUTV_TRY(launch_dgemm(R.L, false, false, lb, b, lb, 1.0, B.Tc, ldc, w.Z, lb, 0.0, w.Z2, lb, nullptr, 0));
    RUTV_TRY(launch_dgemm(R.L, false, false, lb, b, b, -1.0, w.Z2, lb, B.T + l * b * b, b, 0.0, B.Tc + lb * ldc, ldc,
                          nullptr, 0));
  }
  RUTV_TRY(stream_apply_right(R, B.mat, k0 / b, L * b, Wf, rows, B.Tc, ldc, R.Zb, R.Zb2));
  B.k.clear();
  return 0;
}

// queue step k's (W (h x b, ld ldw, rows k:), T, S) of one matrix; flush at G
int defer_uv(HostRun& R, HostRun::Batch& B, i64 k, const double* W, i64 ldw, const double* T, const double* S) {
  const i64 b = R.b, l = (i64)B.k.size();
  const i64 k0 = l == 0 ? k : B.k[0];
  double* Wl = B.W + l * b * B.rows;
  if (k > k0) RUTV_TRY(launch_fill(R.L, k - k0, b, 0.0, Wl + k0, B.rows));
  RUTV_TRY(launch_copy(R.L, B.rows - k, b, W, ldw, Wl + k, B.rows));
  RUTV_TRY(launch_copy(R.L, b, b, T, b, B.T + l * b * b, b));
  RUTV_TRY(launch_copy(R.L, b, b, S, b, B.S + l * b * b, b));
  B.k.push_back(k);
  if ((i64)B.k.size() == R.G) RUTV_TRY(flush_uv(R, B));
  return 0;
}

// One sampled step in 2q + 2 passes over the trailing panels of T (S12):
// the 2q power passes, the S5 read pass (T W_V), and ONE read+write pass that
// applies S5, S7 and the U_s^T fold to each panel and then already takes the
// next step's sample Y' = T(k+b:m, j)^T G' (S1/S2 of step i+1) while the panel
// is resident.  Only step 0 needs a separate S2 pass.
int host_sampled_step(HostRun& R, i64 i) {
  Work& w = R.w;
  // pass directions depend on the step only (not on the history of the call),
  // so a run resumed at step i streams -- and sums -- exactly like one call
  R.dir = (i & 1) == 0;
  const i64 m = R.m, n = R.n, b = R.b, k = i * b, r = m - k, s = n - k;
  const i64 np = R.pc.mats[R.mT].npanels;
  const bool next_sampled = s - b > b;
  // S1 + S2 (step 0 only)
  if (!R.y_ready) {
    RUTV_TRY(launch_gaussian(R.L, R.seed, i, r, b, w.G, r));
    RUTV_TRY(pass(R, R.mT, i, np, false, [&](i64 j, double* X) {
      return launch_dgemm(R.L, true, false, R.pc.width(R.mT, j), b, r, 1.0, X + k, m, w.G, r, 0.0,
                          w.Y + (j - i) * b, s, w.gemm_ws, w.gemm_ws_elems);
    }, k));  // rows above k are not read
  }
  R.y_ready = false;
  // S3
  for (int qq = 0; qq < R.q; ++qq) {
    RUTV_TRY(launch_fill(R.L, r, b, 0.0, w.Z, r));
    RUTV_TRY(pass(R, R.mT, i, np, false, [&](i64 j, double* X) {
      return launch_dgemm(R.L, false, false, r, b, R.pc.width(R.mT, j), 1.0, X + k, m, w.Y + (j - i) * b, s, 1.0,
                          w.Z, r, nullptr, 0);
    }, k));
    RUTV_TRY(pass(R, R.mT, i, np, false, [&](i64 j, double* X) {
      return launch_dgemm(R.L, true, false, R.pc.width(R.mT, j), b, r, 1.0, X + k, m, w.Z, r, 0.0,
                          w.Y + (j - i) * b, s, w.gemm_ws, w.gemm_ws_elems);
    }, k));
  }
  // S4
  RUTV_TRY(panel_qr(R.L, s, b, w.Y, s, w.tauV, w.Wv, s, w.TV, b, w.qw));
  // S5 (read): Z = T(:, k:n) W_V ; Z2 = Z T_V
  RUTV_TRY(launch_fill(R.L, m, b, 0.0, w.Z, m));
  RUTV_TRY(pass(R, R.mT, i, np, false, [&](i64 j, double* X) {
    return launch_dgemm(R.L, false, false, m, b, R.pc.width(R.mT, j), 1.0, X, m, w.Wv + (j - i) * b, s, 1.0, w.Z,
                        m, nullptr, 0);
  }));
  RUTV_TRY(launch_dgemm(R.L, false, false, m, b, b, 1.0, w.Z, m, w.TV, b, 0.0, w.Z2, m, nullptr, 0));
  // panel i: S5 update, S6, S8 and the T part of S9
  {
    double* X;
    RUTV_TRY(R.pc.get(R.mT, i, &X));
    RUTV_TRY(launch_dgemm(R.L, false, true, m, b, b, -1.0, w.Z2, m, w.Wv, s, 1.0, X, m, nullptr, 0));
    RUTV_TRY(panel_qr(R.L, r, b, X + k, m, w.tauU, w.Wu, r, w.TU, b, w.qw));
    RUTV_TRY(launch_triu(R.L, b, b, X + k, m));
    RUTV_TRY(launch_fill(R.L, r - b, b, 0.0, X + k + b, m));
    RUTV_TRY(host_svd_T(R, i, b, X));
    RUTV_TRY(R.pc.put(R.mT, i, true));
  }
  // panels > i (RW): S5 update, S7, U_s^T fold, next step's S2.  apply_left_t
  // uses Z/Z2 as temporaries: keep Z2 (the S5 factor) in Zf meanwhile.
  if (next_sampled) RUTV_TRY(launch_gaussian(R.L, R.seed, i + 1, r - b, b, w.G, r - b));
  RUTV_TRY(launch_copy(R.L, m, b, w.Z2, m, w.Zf, m));
  RUTV_TRY(pass(R, R.mT, i + 1, np, true, [&](i64 j, double* X) {
    const i64 wj = R.pc.width(R.mT, j);
    RUTV_TRY(launch_dgemm(R.L, false, true, m, wj, b, -1.0, w.Zf, m, w.Wv + (j - i) * b, s, 1.0, X, m, nullptr, 0));
    RUTV_TRY(apply_left_t(R.L, w, r, wj, b, X + k, m, w.Wu, r, w.TU, b));
    RUTV_TRY(left_mult_t_inplace(R.L, w.Zv, b, wj, X + k, m, w.Us, b));
    if (!next_sampled) return 0;
    return launch_dgemm(R.L, true, false, wj, b, r - b, 1.0, X + k + b, m, w.G, r - b, 0.0,
                        w.Y + (j - i - 1) * b, s - b, w.gemm_ws, w.gemm_ws_elems);
  }));
  R.y_ready = next_sampled;
  if (R.G > 1) {
    // deferred: merged with the next steps' transforms (flush_uv)
    if (R.mV >= 0) RUTV_TRY(defer_uv(R, R.bv, k, w.Wv, s, w.TV, w.Vs));
    if (R.mU >= 0) RUTV_TRY(defer_uv(R, R.bu, k, w.Wu, r, w.TU, w.Us));
    return 0;
  }
  // V: right transform with W_V; U: right transform with W_U (columns k:m); then their S9 folds
  if (R.mV >= 0) RUTV_TRY(stream_apply_right(R, R.mV, i, b, w.Wv, s, w.TV, b));
  if (R.mU >= 0) RUTV_TRY(stream_apply_right(R, R.mU, i, b, w.Wu, r, w.TU, b));
  return host_fold_uv(R, i, b);
}

int host_final_step(HostRun& R, i64 i) {
  Work& w = R.w;
  const i64 m = R.m, n = R.n, k = i * R.b, r = m - k, s = n - k;
  RUTV_TRY(flush_uv(R, R.bv));
  RUTV_TRY(flush_uv(R, R.bu));
  if (s <= 0) return 0;
  double* X;
  RUTV_TRY(R.pc.get(R.mT, i, &X));
  const bool tall = r > s;
  if (tall) {
    RUTV_TRY(panel_qr(R.L, r, s, X + k, m, w.tauU, w.Wu, r, w.TU, R.b, w.qw));
    RUTV_TRY(launch_triu(R.L, s, s, X + k, m));
    RUTV_TRY(launch_fill(R.L, r - s, s, 0.0, X + k + s, m));
  }
  RUTV_TRY(host_svd_T(R, i, s, X));
  RUTV_TRY(R.pc.put(R.mT, i, true));
  if (tall && R.mU >= 0) RUTV_TRY(stream_apply_right(R, R.mU, i, s, w.Wu, r, w.TU, R.b));
  return host_fold_uv(R, i, s);
}

// ---------------------------------------------------------------------------
// Sharded + host-streamed: the rank's block-cyclic
// columns of A (dist.cu's layout) live in host memory and stream through the
// rank's device panel cache; U and V are the rank's row ranges, streamed by
// column panels.  One step is host_sampled_step's pass structure with dist.cu's
// collectives: the local sample passes with an AllReduce of Z per power step,
// the AllGather of Y and the same QR(Y) on every rank, the T W_V read pass +
// AllReduce, the owner's panel (S5, S6, SVD, T11 = diag d, A01 V_s), ONE
// broadcast of [W_U | T_U | U_s | V_s], and the read-write pass over the
// rank's later panels (S5, S7, the U_s^T fold, the next step's local sample).

int hd_sampled_step(HostRun& R, i64 i) {
  Work& w = R.w;
  const Layout& lay = R.lay;
  const int p = lay.p, P = lay.P, o = (int)(i % P);
  const i64 m = R.m, n = R.n, b = R.b, k = i * b, r = m - k, s = n - k;
  const i64 np = R.pc.mats[R.mT].npanels;
  const i64 lp0 = lay.lb_before(p, i), lp1 = lay.lb_before(p, i + 1);
  const i64 sl = lay.ncols(p) - lp0 * b, maxs = R.maxs;
  const bool next_sampled = s - b > b;
  cudaStream_t st = R.L.stream;
  R.dir = (i & 1) == 0;
  // S1 + S2 (the first step; afterwards taken by the previous RW pass)
  if (!R.y_ready) {
    RUTV_TRY(launch_gaussian(R.L, R.seed, i, r, b, w.G, r));
    RUTV_TRY(pass(R, R.mT, lp0, np, false, [&](i64 j, double* X) {
      return launch_dgemm(R.L, true, false, R.pc.width(R.mT, j), b, r, 1.0, X + k, m, w.G, r, 0.0,
                          R.Yl + (j - lp0) * b, maxs, w.gemm_ws, w.gemm_ws_elems);
    }, k));
  }
  R.y_ready = false;
  // S3: Z = sum_p A_p Y_p (AllReduce); Y_p = A_p^T Z
  for (int qq = 0; qq < R.q; ++qq) {
    RUTV_TRY(launch_fill(R.L, r, b, 0.0, w.Z, r));
    RUTV_TRY(pass(R, R.mT, lp0, np, false, [&](i64 j, double* X) {
      return launch_dgemm(R.L, false, false, r, b, R.pc.width(R.mT, j), 1.0, X + k, m, R.Yl + (j - lp0) * b, maxs,
                          1.0, w.Z, r, nullptr, 0);
    }, k));
    RUTV_TRY(R.comm->allreduce_sum(w.Z, r * b, st));
    RUTV_TRY(pass(R, R.mT, lp0, np, false, [&](i64 j, double* X) {
      return launch_dgemm(R.L, true, false, R.pc.width(R.mT, j), b, r, 1.0, X + k, m, w.Z, r, 0.0,
                          R.Yl + (j - lp0) * b, maxs, w.gemm_ws, w.gemm_ws_elems);
    }, k));
  }
  // S4: Y in global order, the same QR on every rank; this rank's rows of W_V
  RUTV_TRY(R.comm->allgather(R.Yl, R.Yall, maxs * b, st));
  RUTV_TRY(launch_cyclic_gather_rows(R.L, s, b, k, b, P, i, R.Yall, maxs, maxs * b, w.Y, s));
  RUTV_TRY(panel_qr(R.L, s, b, w.Y, s, w.tauV, w.Wv, s, w.TV, b, w.qw));
  RUTV_TRY(launch_cyclic_scatter_rows(R.L, sl, b, k, b, P, p, lp0, w.Wv, s, R.Wl, maxs));
  // S5 (read): Z = sum_p T_p W_p (all m rows, AllReduce); Z2 = Z T_V
  RUTV_TRY(launch_fill(R.L, m, b, 0.0, w.Z, m));
  RUTV_TRY(pass(R, R.mT, lp0, np, false, [&](i64 j, double* X) {
    return launch_dgemm(R.L, false, false, m, b, R.pc.width(R.mT, j), 1.0, X, m, R.Wl + (j - lp0) * b, maxs, 1.0,
                        w.Z, m, nullptr, 0);
  }));
  RUTV_TRY(R.comm->allreduce_sum(w.Z, m * b, st));
  RUTV_TRY(launch_dgemm(R.L, false, false, m, b, b, 1.0, w.Z, m, w.TV, b, 0.0, w.Z2, m, nullptr, 0));
  // the owner's panel i: S5 update, S6, S8, T11 = diag d, A01 V_s
  double* Wu = R.wbuf;
  double* TU = Wu + r * b;
  double* Us = TU + b * b;
  double* Vs = Us + b * b;
  if (p == o) {
    double* X;
    RUTV_TRY(R.pc.get(R.mT, lp0, &X));
    RUTV_TRY(launch_dgemm(R.L, false, true, m, b, b, -1.0, w.Z2, m, R.Wl, maxs, 1.0, X, m, nullptr, 0));
    RUTV_TRY(panel_qr(R.L, r, b, X + k, m, w.tauU, Wu, r, TU, b, w.qw));
    RUTV_TRY(launch_triu(R.L, b, b, X + k, m));
    RUTV_TRY(launch_fill(R.L, r - b, b, 0.0, X + k + b, m));
    RUTV_TRY(launch_jacobi_svd(R.L, b, X + k, m, Us, w.d, Vs, w.status, (int)(i + 1), w.jac, w.jac_elems));
    RUTV_TRY(launch_set_diag(R.L, b, w.d, X + k, m));
    RUTV_TRY(right_mult_inplace(R.L, w.Zf, k, b, X, m, Vs, b));  // A01 V_s
    RUTV_TRY(R.pc.put(R.mT, lp0, true));
  }
  RUTV_TRY(R.comm->bcast(R.wbuf, r * b + 3 * b * b, o, st));
  RUTV_TRY(launch_copy(R.L, b, b, Us, b, w.Us, b));
  RUTV_TRY(launch_copy(R.L, b, b, Vs, b, w.Vs, b));
  // the rank's later panels (RW): S5, S7, U_s^T fold, the next step's local sample
  if (next_sampled) RUTV_TRY(launch_gaussian(R.L, R.seed, i + 1, r - b, b, w.G, r - b));
  RUTV_TRY(launch_copy(R.L, m, b, w.Z2, m, w.Zf, m));
  RUTV_TRY(pass(R, R.mT, lp1, np, true, [&](i64 j, double* X) {
    const i64 wj = R.pc.width(R.mT, j);
    RUTV_TRY(launch_dgemm(R.L, false, true, m, wj, b, -1.0, w.Zf, m, R.Wl + (j - lp0) * b, maxs, 1.0, X, m, nullptr,
                          0));
    RUTV_TRY(apply_left_t(R.L, w, r, wj, b, X + k, m, Wu, r, TU, b));
    RUTV_TRY(left_mult_t_inplace(R.L, w.Zv, b, wj, X + k, m, w.Us, b));
    if (!next_sampled) return 0;
    return launch_dgemm(R.L, true, false, wj, b, r - b, 1.0, X + k + b, m, w.G, r - b, 0.0, R.Yl + (j - lp1) * b,
                        maxs, w.gemm_ws, w.gemm_ws_elems);
  }));
  R.y_ready = next_sampled;
  if (R.G > 1) {
    if (R.mV >= 0) RUTV_TRY(defer_uv(R, R.bv, k, w.Wv, s, w.TV, w.Vs));
    if (R.mU >= 0) RUTV_TRY(defer_uv(R, R.bu, k, Wu, r, TU, w.Us));
    return 0;
  }
  if (R.mV >= 0) RUTV_TRY(stream_apply_right(R, R.mV, i, b, w.Wv, s, w.TV, b));
  if (R.mU >= 0) RUTV_TRY(stream_apply_right(R, R.mU, i, b, Wu, r, TU, b));
  return host_fold_uv(R, i, b);
}

int hd_final_step(HostRun& R, i64 i) {
  Work& w = R.w;
  const Layout& lay = R.lay;
  const int p = lay.p, o = (int)(i % lay.P);
  const i64 m = R.m, n = R.n, k = i * R.b, r = m - k, s = n - k;
  RUTV_TRY(flush_uv(R, R.bv));
  RUTV_TRY(flush_uv(R, R.bu));
  if (s <= 0) return 0;
  const bool tall = r > s;
  double* Wu = R.wbuf;
  double* TU = Wu + r * s;
  double* Us = TU + s * s;
  double* Vs = Us + s * s;
  if (p == o) {
    double* X;
    const i64 lp = lay.lb_before(p, i);
    RUTV_TRY(R.pc.get(R.mT, lp, &X));
    if (tall) {
      RUTV_TRY(panel_qr(R.L, r, s, X + k, m, w.tauU, Wu, r, TU, s, w.qw));
      RUTV_TRY(launch_triu(R.L, s, s, X + k, m));
      RUTV_TRY(launch_fill(R.L, r - s, s, 0.0, X + k + s, m));
    }
    RUTV_TRY(launch_jacobi_svd(R.L, s, X + k, m, Us, w.d, Vs, w.status, (int)(i + 1), w.jac, w.jac_elems));
    RUTV_TRY(launch_set_diag(R.L, s, w.d, X + k, m));
    RUTV_TRY(right_mult_inplace(R.L, w.Zf, k, s, X, m, Vs, s));  // A01 V_s
    RUTV_TRY(R.pc.put(R.mT, lp, true));
  }
  RUTV_TRY(R.comm->bcast(R.wbuf, r * s + 3 * s * s, o, R.L.stream));
  RUTV_TRY(launch_copy(R.L, s, s, Us, s, w.Us, s));
  RUTV_TRY(launch_copy(R.L, s, s, Vs, s, w.Vs, s));
  if (tall && R.mU >= 0) RUTV_TRY(stream_apply_right(R, R.mU, i, s, Wu, r, TU, s));
  return host_fold_uv(R, i, s);
}

}  // namespace

}  // namespace rutv

using namespace rutv;

extern "C" {

static int factor_host_impl(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b, int q,
                            uint64_t seed, unsigned flags, size_t device_cache_bytes, double* U_host, int64_t ldu,
                            double* V_host, int64_t ldv, int64_t step_begin, int64_t step_end,
                            randutv_host_report* report, Comm* comm = nullptr);

}  // extern "C"

namespace rutv {
// the sharded host-streamed entry used by randutv_factor_dist_host and its
// loopback harness (dist.cu): the rank's columns / rows in host memory
int dist_host_factor(randutv_ctx* ctx, Comm* comm, int64_t m, int64_t n, double* A_local, int64_t lda, int64_t b, int q,
                     uint64_t seed, unsigned flags, size_t cache_bytes, double* U_local, int64_t ldu,
                     double* V_local, int64_t ldv, randutv_host_report* report) {
  return factor_host_impl(ctx, m, n, A_local, lda, b, q, seed, flags, cache_bytes, U_local, ldu, V_local, ldv, 0,
                          INT64_MAX, report, comm);
}
}  // namespace rutv

extern "C" {

RANDUTV_API int randutv_factor_dist_host(randutv_ctx* ctx, int64_t m, int64_t n, double* A_local_host, int64_t lda,
                                         int64_t b, int q, uint64_t seed, unsigned flags, size_t device_cache_bytes,
                                         double* U_local_host, int64_t ldu, double* V_local_host, int64_t ldv,
                                         randutv_host_report* report) {
  RUTV_TRY(begin_call(ctx));
  if (!ctx->comm) return RANDUTV_ERR_NOCOMM;
  return dist_host_factor(ctx, ctx->comm, m, n, A_local_host, lda, b, q, seed, flags, device_cache_bytes,
                          U_local_host, ldu, V_local_host, ldv, report);
}

RANDUTV_API int randutv_factor_host(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b,
                                    int q, uint64_t seed, unsigned flags, size_t device_cache_bytes, double* U_host,
                                    int64_t ldu, double* V_host, int64_t ldv, randutv_host_report* report) {
  return factor_host_impl(ctx, m, n, A_host, lda, b, q, seed, flags, device_cache_bytes, U_host, ldu, V_host, ldv, 0,
                          INT64_MAX, report);
}

RANDUTV_API int randutv_factor_host_steps(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda,
                                          int64_t b, int q, uint64_t seed, unsigned flags, size_t device_cache_bytes,
                                          double* U_host, int64_t ldu, double* V_host, int64_t ldv,
                                          int64_t step_begin, int64_t step_end, randutv_host_report* report) {
  if (step_begin < 0) return -15;
  if (step_end <= step_begin) return -16;
  return factor_host_impl(ctx, m, n, A_host, lda, b, q, seed, flags, device_cache_bytes, U_host, ldu, V_host, ldv,
                          step_begin, step_end, report);
}

static int factor_host_impl(randutv_ctx* ctx, int64_t m, int64_t n, double* A_host, int64_t lda, int64_t b, int q,
                            uint64_t seed, unsigned flags, size_t device_cache_bytes, double* U_host, int64_t ldu,
                            double* V_host, int64_t ldv, int64_t step_begin, int64_t step_end,
                            randutv_host_report* report, Comm* comm) {
  RUTV_TRY(begin_call(ctx));
  const bool uv = !(flags & RANDUTV_NO_UV);
  // sharded: the rank's layout (dist.cu) -- its columns of A, rows of U and V
  const int P = comm ? comm->nranks : 1, prank = comm ? comm->rank : 0;
  const i64 bb = std::max<i64>(1, std::min<i64>(b, n));
  Layout lay{m, n, bb, P, prank, (n + bb - 1) / bb};
  const i64 ncl = lay.ncols(prank);
  const i64 u0 = Layout::row0(m, P, prank), mu = Layout::row0(m, P, prank + 1) - u0;
  const i64 v0 = Layout::row0(n, P, prank), nv = Layout::row0(n, P, prank + 1) - v0;
  int local = 0;
  if (flags & RANDUTV_REORTH) local = -9;  // not implemented on the host-streamed path
  else if (ctx->oversample > 0) local = -9;  // nor is oversampling (RANDUTV_OPT_OVERSAMPLE)
  else if (comm && (flags & (RANDUTV_CHECK_FINITE | RANDUTV_ASYNC))) local = -9;
  else if (n < 1) local = -3;
  else if (m < n) local = -2;
  else if (!A_host && ncl > 0) local = -4;
  else if (lda < m) local = -5;
  else if (b < 1) local = -6;
  else if (q < 0) local = -7;
  else if (uv && !U_host && mu > 0) local = -11;
  else if (uv && ldu < std::max<i64>(comm ? mu : m, 1)) local = -12;
  else if (uv && !V_host && nv > 0) local = -13;
  else if (uv && ldv < std::max<i64>(comm ? nv : n, 1)) local = -14;
  // every rank's verdict (arguments here, workspace below) is agreed before
  // the first collective of a sharded call (dist.cu's agreement)
  auto agree = [&](int loc) -> int {
    if (!comm) return loc;
    if (!comm->dflag && cudaMalloc(&comm->dflag, sizeof(int)) != cudaSuccess) return RANDUTV_ERR_ALLOC;
    int h = loc == 0 ? 1 : 0;
    RUTV_CUDA(cudaMemcpyAsync(comm->dflag, &h, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    RUTV_TRY(comm->allreduce_min_int(comm->dflag, 1, ctx->stream));
    RUTV_CUDA(cudaMemcpyAsync(&h, comm->dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RUTV_TRY(comm->sync(ctx->stream));
    if (loc != 0) return loc;
    return h ? 0 : RANDUTV_ERR_PEER;
  };
  if (local != 0) return agree(local);
  randutv_host_report rep;
  memset(&rep, 0, sizeof(rep));

  HostRun R;
  R.ctx = ctx;
  R.L = ctx->launch();
  R.m = m;
  R.n = n;
  R.b = bb;
  R.q = q;
  R.seed = seed;
  R.pc.b = bb;
  R.pc.rep = &rep;
  R.pc.slot_elems = ((std::max(m, n) * bb + 31) / 32) * 32;
  R.comm = comm;
  R.lay = lay;
  R.maxs = std::max<i64>(lay.max_trailing(0), 1);
  // workspace: the in-HBM driver's buffers + U_s of the deferred fold + the slots
  Carver dry{nullptr, 0, 0, true};
  {
    const char* e = getenv("RUTV_HOST_UV_BATCH");
    R.G = uv ? (e ? atoi(e) : 8) : 1;
    if (R.G < 1) R.G = 1;
  }
  const i64 Gb = R.G * bb, mx = std::max(m, n);
  auto carve_batch = [&](Carver& c) {
    if (R.G <= 1) return;
    R.bu.W = c.take<double>(m * Gb);
    R.bv.W = c.take<double>(n * Gb);
    for (HostRun::Batch* B : {&R.bu, &R.bv}) {
      B->T = c.take<double>(Gb * bb);
      B->S = c.take<double>(Gb * bb);
      B->Tc = c.take<double>(Gb * Gb);
    }
    R.Zb = c.take<double>(mx * Gb);
    R.Zb2 = c.take<double>(mx * Gb);
  };
  auto carve_dist = [&](Carver& c) {
    if (!comm) return;
    R.Yl = c.take<double>(R.maxs * bb);
    R.Yall = c.take<double>((i64)P * R.maxs * bb);
    R.Wl = c.take<double>(R.maxs * bb);
    R.wbuf = c.take<double>(m * bb + 3 * bb * bb);
  };
  carve(dry, R.w, m, n, bb, 0, false);
  carve_batch(dry);
  carve_dist(dry);
  const size_t fixed = dry.off;
  const size_t slot_bytes = (size_t)R.pc.slot_elems * 8;
  size_t budget = device_cache_bytes;
  if (budget == 0) {
    size_t fr = 0, tot = 0;
    RUTV_CUDA(cudaMemGetInfo(&fr, &tot));
    budget = fr / 2;
  }
  i64 nslots = (i64)(budget / slot_bytes);
  const i64 npT = (ncl + bb - 1) / bb, npU = uv ? (m + bb - 1) / bb : 0, npV = uv ? (n + bb - 1) / bb : 0;
  nslots = std::min<i64>(nslots, npT + npU + npV);
  if (nslots < 3) nslots = 3;
  {
    const int ws_st = fault_alloc(comm ? comm->rank : -1) && comm ? RANDUTV_ERR_ALLOC
                                                                  : ensure_ws(ctx, fixed + (size_t)nslots * slot_bytes + kAlign);
    RUTV_TRY(agree(ws_st));
  }
  Carver real{(char*)ctx->ws, 0, ctx->ws_bytes, false};
  carve(real, R.w, m, n, bb, 0, false);
  carve_batch(real);
  carve_dist(real);
  double* slots = real.take<double>(nslots * R.pc.slot_elems);
  rep.cache_slots = nslots;
  rep.slot_bytes = (int64_t)slot_bytes;

  // pin the host matrices for the duration of the call if the caller did not
  std::vector<void*> registered;
  auto pin = [&](double* h, i64 ld, i64 cols) -> int {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) == cudaSuccess && a.type == cudaMemoryTypeHost) return 0;
    cudaGetLastError();
    RUTV_CUDA(cudaHostRegister(h, (size_t)ld * cols * 8, cudaHostRegisterDefault));
    registered.push_back(h);
    return 0;
  };
  int st = ncl > 0 ? pin(A_host, lda, ncl) : 0;
  if (st == 0 && uv && mu > 0) st = pin(U_host, ldu, m);
  if (st == 0 && uv && nv > 0) st = pin(V_host, ldv, n);

  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (st == 0 && (cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) != cudaSuccess ||
                  cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) != cudaSuccess ||
                  cudaEventCreate(&t0) != cudaSuccess || cudaEventCreate(&t1) != cudaSuccess))
    st = RANDUTV_ERR_CUDA;
  if (st == 0) {
    R.pc.comp = ctx->stream;
    R.pc.h2d = h2d;
    R.pc.d2h = d2h;
    R.pc.timer.on = report != nullptr;
    st = R.pc.init(nslots, slots);
  }
  // sharded: a rank that failed to pin or to set up its streams must not leave
  // the others waiting in the first collective
  if (comm) st = agree(st);
  if (st == 0) {
    R.mT = R.pc.add_mat(A_host, m, ncl, lda);  // all of A, or the rank's columns
    if (uv && mu > 0) {
      R.mU = R.pc.add_mat(U_host, comm ? mu : m, m, ldu);  // all of U, or the rank's rows
      R.bu.mat = R.mU;
      R.bu.rows = m;
    }
    if (uv && nv > 0) {
      R.mV = R.pc.add_mat(V_host, comm ? nv : n, n, ldv);
      R.bv.mat = R.mV;
      R.bv.rows = n;
    }
    cudaEventRecord(t0, ctx->stream);
    st = start_status(ctx, R.w);
  }
  const i64 nsamp = sampled_steps(n, bb);
  if (st == 0 && step_begin > nsamp) st = -15;  // past the final step
  // U := I, V := I panel by panel on the device (no host traffic in); a
  // resumed range (step_begin > 0) continues from the U, V in host memory
  if (st == 0 && uv && step_begin == 0) {
    for (int mat : {R.mU, R.mV}) {
      if (mat < 0) continue;
      const HostMat& M = R.pc.mats[mat];
      const i64 row0 = !comm ? 0 : (mat == R.mU ? u0 : v0);  // global row of the panel's first row
      for (i64 j = 0; j < M.npanels && st == 0; ++j) {
        double* X;
        st = R.pc.get(mat, j, &X, false);
        if (st == 0) st = launch_set_identity_shift(R.L, M.rows, R.pc.width(mat, j), j * bb - row0, X, M.rows);
        if (st == 0) st = R.pc.put(mat, j, true);
      }
    }
  }
  if (st == 0 && (flags & RANDUTV_CHECK_FINITE)) {
    // scan panel by panel through the cache
    st = cudaMemsetAsync(R.w.flag, 0, sizeof(int), ctx->stream) == cudaSuccess ? 0 : RANDUTV_ERR_CUDA;
    for (i64 j = 0; j < npT && st == 0; ++j) {
      double* X;
      st = R.pc.get(R.mT, j, &X);
      if (st == 0) st = launch_nonfinite(R.L, m, R.pc.width(R.mT, j), X, m, R.w.flag);
      if (st == 0) st = R.pc.put(R.mT, j, false);
    }
    int flag = 0;
    if (st == 0 && (cudaMemcpyAsync(&flag, R.w.flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) !=
                        cudaSuccess ||
                    cudaStreamSynchronize(ctx->stream) != cudaSuccess))
      st = RANDUTV_ERR_CUDA;
    if (st == 0 && flag) st = RANDUTV_ERR_NONFINITE;
  }
  if (st == 0) {
    // Belady eviction for T-only runs without the finiteness scan (their T
    // access sequence is exactly the plan)
    if (!comm && !uv && !(flags & RANDUTV_CHECK_FINITE) && belady_on()) {
      build_plan(n, bb, q, nsamp, step_begin, step_end, R.pc.plan, R.pc.nxt);
      R.pc.plan_mat = R.mT;
      R.pc.cursor = 0;
      R.pc.use_plan = true;
    }
    const i64 last = std::min<i64>(step_end, nsamp);
    for (i64 i = step_begin; i < last && st == 0; ++i) st = comm ? hd_sampled_step(R, i) : host_sampled_step(R, i);
    if (st == 0 && step_end > nsamp) st = comm ? hd_final_step(R, nsamp) : host_final_step(R, nsamp);
    // a range that stops before the final step leaves no deferred U / V
    // transform behind: the host U, V are the state after step last - 1
    if (st == 0 && step_end <= nsamp) st = flush_uv(R, R.bv);
    if (st == 0 && step_end <= nsamp) st = flush_uv(R, R.bu);
    if (st == 0) st = R.pc.flush();
    if (st == 0) {
      // the compute stream must not return before the write-backs land
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(e, d2h);
        cudaStreamWaitEvent(ctx->stream, e, 0);
        cudaEventRecord(e, h2d);
        cudaStreamWaitEvent(ctx->stream, e, 0);
        cudaEventDestroy(e);
      }
      cudaEventRecord(t1, ctx->stream);
      if (comm) {
        // every rank returns the first non-converged block; waits through the communicator
        st = comm->allreduce_min_int(R.w.status, 1, ctx->stream);
        if (st == 0) st = comm->sync(ctx->stream);
      }
      if (st == 0) st = finish(ctx, R.w);
    }
  }
  {
    float ms = 0.f;
    if (t0 && t1 && cudaEventElapsedTime(&ms, t0, t1) == cudaSuccess) rep.wall_ms = ms;
    auto sum = [&](const std::vector<std::pair<size_t, size_t>>& v) {
      double tot = 0.0;
      for (auto& pr : v) {
        float x = 0.f;
        if (cudaEventElapsedTime(&x, R.pc.timer.pool[pr.first], R.pc.timer.pool[pr.second]) == cudaSuccess) tot += x;
      }
      return tot;
    };
    rep.h2d_ms = sum(R.pc.timer.h2d);
    rep.d2h_ms = sum(R.pc.timer.d2h);
  }
  cudaStreamSynchronize(ctx->stream);
  if (h2d) cudaStreamSynchronize(h2d);
  if (d2h) cudaStreamSynchronize(d2h);
  R.pc.destroy();
  if (h2d) cudaStreamDestroy(h2d);
  if (d2h) cudaStreamDestroy(d2h);
  if (t0) cudaEventDestroy(t0);
  if (t1) cudaEventDestroy(t1);
  for (void* p : registered) cudaHostUnregister(p);
  cudaGetLastError();
  ctx->stats.h2d_bytes += rep.h2d_bytes;
  ctx->stats.d2h_bytes += rep.d2h_bytes;
  if (report) *report = rep;
  if (st == 0) ctx->stats.factorizations++;
  return st;
}

}  // extern "C"
