"""Python binding of librandutv.so (include/randutv.h) -- argument marshalling only.

Every arithmetic step of randUTV runs in the CUDA kernels of the shared
library; this module only converts torch tensors / numpy arrays into pointers,
leading dimensions and the ctx stream, and raises on a non-zero status.  There
is no CPU fallback: if the library is missing, importing a compute function
raises.

Column-major convention: a column-major m x n FP64 matrix on the device is a
torch tensor of shape (m, n) with strides (1, ld), e.g. ``colmajor(m, n)``.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RUTV_LIB", os.path.join(_HERE, "librandutv.so"))  # RUTV_LIB: A/B variants only

RANDUTV_NO_UV = 1
RANDUTV_CHECK_FINITE = 2
RANDUTV_REORTH = 4
RANDUTV_ASYNC = 8
RANDUTV_ECON_U = 16
RANDUTV_OPT_JACOBI_SWEEPS = 1
RANDUTV_OPT_OVERSAMPLE = 2
RANDUTV_ERR_BASE = 0x40000000
RANDUTV_ERR_CUDA = RANDUTV_ERR_BASE + 0
RANDUTV_ERR_ALLOC = RANDUTV_ERR_BASE + 1
RANDUTV_ERR_NONFINITE = RANDUTV_ERR_BASE + 2
RANDUTV_ERR_CTX = RANDUTV_ERR_BASE + 3
RANDUTV_ERR_NCCL = RANDUTV_ERR_BASE + 4
RANDUTV_ERR_NOCOMM = RANDUTV_ERR_BASE + 5
RANDUTV_ERR_PEER = RANDUTV_ERR_BASE + 6
RANDUTV_UNIQUE_ID_BYTES = 128

# name -> (restype, argtypes) ; mirrors include/randutv.h
_i64, _u64, _int, _uint, _dbl, _vp = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint,
                                      ctypes.c_double, ctypes.c_void_p)


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("factorizations", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64),
                ("d2h_bytes", ctypes.c_int64)]


class Profile(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("ms", ctypes.c_double), ("flops", ctypes.c_double),
                ("bytes", ctypes.c_double), ("busy_ms", ctypes.c_double)]


class HostReport(ctypes.Structure):
    _fields_ = [("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64), ("cache_hits", ctypes.c_int64),
                ("cache_misses", ctypes.c_int64), ("cache_slots", ctypes.c_int64), ("slot_bytes", ctypes.c_int64),
                ("wall_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double), ("d2h_ms", ctypes.c_double)]


PROF_KINDS = {"dgemm": 0, "qr_leaf": 1, "jacobi": 2, "gaussian": 3, "fold_wait": 4}

SIGNATURES = {
    "randutv_create": (_int, [ctypes.POINTER(_vp), _int, _vp]),
    "randutv_destroy": (_int, [_vp]),
    "randutv_set_stream": (_int, [_vp, _vp]),
    "randutv_set_option": (_int, [_vp, _int, _i64]),
    "randutv_workspace_bytes": (_int, [_i64, _i64, _i64, _int, _uint, ctypes.POINTER(ctypes.c_size_t)]),
    "randutv_factor": (_int, [_i64, _i64, _vp, _i64, _i64, _int, _u64, _vp, _vp, _vp]),
    "randutv_factor_ex": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _int, _u64, _uint,
                                 _vp, _i64, _vp, _i64, _vp, _i64]),
    "randutv_factor_rank": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _i64, _int, _u64, _uint,
                                   _vp, _i64, _vp, _i64, _vp, _i64, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]),
    "randutv_factor_tol": (_int, [_vp, _i64, _i64, _vp, _i64, _dbl, _i64, _int, _u64, _uint, _vp, _i64, _vp, _i64,
                                  _vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_dbl)]),
    "randutv_hqrrp": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _u64, _uint, _vp, _vp, _i64]),
    "randutv_hqrrp_rank": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _i64, _u64, _uint, _vp, _vp, _i64,
                                  ctypes.POINTER(_dbl)]),
    "randutv_hqrrp_host": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _u64, _uint, _vp, _vp, ctypes.POINTER(HostReport)]),
    "randutv_wait": (_int, [_vp]),
    "randutv_status_string": (ctypes.c_char_p, [_int]),
    "randutv_last_error": (ctypes.c_char_p, []),
    "randutv_get_stats": (_int, [_vp, ctypes.POINTER(Stats)]),
    "randutv_reset_stats": (_int, [_vp]),
    "randutv_set_profiling": (_int, [_vp, _int]),
    "randutv_get_profile": (_int, [_vp, _int, ctypes.POINTER(Profile)]),
    "randutv_gaussian": (_int, [_vp, _u64, _i64, _i64, _i64, _vp, _i64]),
    "randutv_dgemm": (_int, [_vp, _int, _int, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64]),
    "randutv_dgemm_plan": (_int, [_i64, _i64, _i64, _i64, _int, _int, ctypes.POINTER(ctypes.c_int64)]),
    "randutv_panel_qr": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _i64]),
    "randutv_small_svd": (_int, [_vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "randutv_factor_host": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _int, _u64, _uint, ctypes.c_size_t, _vp, _i64,
                                   _vp, _i64, ctypes.POINTER(HostReport)]),
    "randutv_factor_host_steps": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _int, _u64, _uint, ctypes.c_size_t, _vp,
                                         _i64, _vp, _i64, _i64, _i64, ctypes.POINTER(HostReport)]),
    "randutv_factor_dist_host": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _int, _u64, _uint, ctypes.c_size_t, _vp,
                                        _i64, _vp, _i64, ctypes.POINTER(HostReport)]),
    "randutv_factor_dist_host_loopback": (_int, [_int, _int, _i64, _i64, ctypes.POINTER(_vp), _i64, _i64, _int, _u64,
                                                 _uint, ctypes.c_size_t, ctypes.POINTER(_vp), _i64,
                                                 ctypes.POINTER(_vp), _i64]),
    "randutv_dist_layout": (_int, [_i64, _i64, _i64, _int, _int, ctypes.POINTER(_i64)]),
    "randutv_nccl_unique_id": (_int, [_vp]),
    "randutv_comm_init": (_int, [_vp, _vp, _int, _int]),
    "randutv_factor_dist": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _int, _u64, _uint, _vp, _i64, _vp, _i64]),
    "randutv_factor_dist_rank": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _i64, _int, _u64, _uint, _vp, _i64, _vp,
                                        _i64, ctypes.POINTER(_dbl)]),
    "randutv_factor_dist_loopback": (_int, [_int, _int, _i64, _i64, ctypes.POINTER(_vp), _i64, _i64, _int, _u64,
                                            _uint, ctypes.POINTER(_vp), _i64, ctypes.POINTER(_vp), _i64, _i64,
                                            ctypes.POINTER(_dbl)]),
}

_lib = None


def load_library(path=LIB_PATH):
    """Load librandutv.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class RandUTVError(RuntimeError):
    def __init__(self, fn, status):
        lib = load_library()
        msg = lib.randutv_status_string(status).decode()
        if status == RANDUTV_ERR_CUDA:
            msg += ": " + lib.randutv_last_error().decode()
        super().__init__(f"{fn} returned {status} ({msg})")
        self.status = status


def _check(fn, status, allow_positive=False):
    if status != 0 and not (allow_positive and 0 < status < RANDUTV_ERR_BASE):
        raise RandUTVError(fn, status)
    return status


# ----------------------------------------------------------------------------- tensors

def colmajor(m, n, device="cuda", fill=None):
    """Column-major m x n float64 tensor (shape (m, n), strides (1, m))."""
    import torch
    t = torch.empty((n, m), dtype=torch.float64, device=device).t()
    if fill is not None:
        t.fill_(fill)
    return t


def as_colmajor(X):
    """Column-major copy (or the tensor itself if already column-major with ld >= rows)."""
    import torch
    m, n = X.shape
    if X.dtype == torch.float64 and X.stride(0) == 1 and X.stride(1) >= max(m, 1):
        return X
    Y = colmajor(m, n, device=X.device)
    Y.copy_(X)
    return Y


def _ld(X):
    if X.dim() != 2 or X.stride(0) != 1:
        raise ValueError("expected a column-major 2-D float64 tensor (stride(0) == 1)")
    return max(X.stride(1), 1) if X.shape[1] > 1 else max(X.shape[0], 1)


def _ptr(X):
    return ctypes.c_void_p(X.data_ptr()) if X is not None else None


class Context:
    """A randutv_ctx bound to a CUDA device and stream (torch's current stream by default)."""

    def __init__(self, device=None, stream=None):
        import torch
        self.lib = load_library()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        h = ctypes.c_void_p()
        _check("randutv_create", self.lib.randutv_create(ctypes.byref(h), self.device,
                                                          ctypes.c_void_p(stream.cuda_stream)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.randutv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, option, value):
        _check("randutv_set_option", self.lib.randutv_set_option(self.h, int(option), int(value)))

    def stats(self):
        s = Stats()
        _check("randutv_get_stats", self.lib.randutv_get_stats(self.h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def reset_stats(self):
        _check("randutv_reset_stats", self.lib.randutv_reset_stats(self.h))

    def set_profiling(self, on=True):
        _check("randutv_set_profiling", self.lib.randutv_set_profiling(self.h, 1 if on else 0))

    def profile(self):
        out = {}
        for name, kind in PROF_KINDS.items():
            p = Profile()
            _check("randutv_get_profile", self.lib.randutv_get_profile(self.h, kind, ctypes.byref(p)))
            out[name] = {k: getattr(p, k) for k, _ in Profile._fields_}
        return out

    # ---------------------------------------------------------------- factorisations
    def randutv_factor_ex(self, A, b, q, seed, build_uv=True, U=None, T=None, V=None, flags=0,
                          allow_nonconvergence=False, econ_u=False):
        """Full randUTV of the column-major device matrix A: returns (U, T, V, status).
        econ_u: U is the economy m x n factor (RANDUTV_ECON_U)."""
        m, n = A.shape
        if not build_uv:
            flags |= RANDUTV_NO_UV
        if econ_u:
            flags |= RANDUTV_ECON_U
        if T is None:
            T = colmajor(m, n, device=A.device)
        if build_uv:
            U = colmajor(m, n if econ_u else m, device=A.device) if U is None else U
            V = colmajor(n, n, device=A.device) if V is None else V
        st = self.lib.randutv_factor_ex(self.h, m, n, _ptr(A), _ld(A), int(b), int(q), int(seed) & (2**64 - 1),
                                        flags, _ptr(U), _ld(U) if U is not None else 1, _ptr(T), _ld(T),
                                        _ptr(V), _ld(V) if V is not None else 1)
        _check("randutv_factor_ex", st, allow_positive=allow_nonconvergence)
        return U, T, V, st

    def wait(self):
        """Synchronise; the status of the last RANDUTV_ASYNC factorisation."""
        st = self.lib.randutv_wait(self.h)
        _check("randutv_wait", st, allow_positive=True)
        return st

    def randutv_factor_rank(self, A, k, b, q, seed, build_uv=True, flags=0, resid_2=False):
        """Truncated randUTV: returns (Uk, Tk, V, rho), or (Uk, Tk, V, rho, rho_2) with
        resid_2 (the spectral-norm residual, reading A11)."""
        m, n = A.shape
        if not build_uv:
            flags |= RANDUTV_NO_UV
        Tk = colmajor(k, n, device=A.device)
        Uk = colmajor(m, k, device=A.device) if build_uv else None
        V = colmajor(n, n, device=A.device) if build_uv else None
        rho = ctypes.c_double()
        rho2 = ctypes.c_double()
        st = self.lib.randutv_factor_rank(self.h, m, n, _ptr(A), _ld(A), int(k), int(b), int(q),
                                          int(seed) & (2**64 - 1), flags, _ptr(Uk), _ld(Uk) if Uk is not None else 1,
                                          _ptr(Tk), _ld(Tk), _ptr(V), _ld(V) if V is not None else 1,
                                          ctypes.byref(rho), ctypes.byref(rho2) if resid_2 else None)
        _check("randutv_factor_rank", st)
        if resid_2:
            return Uk, Tk, V, rho.value, rho2.value
        return Uk, Tk, V, rho.value

    def randutv_factor_tol(self, A, tol, b, q, seed, build_uv=True, flags=0):
        """Adaptive-rank randUTV: returns (Uk, Tk, V, rho, k) for the first k = i*b whose
        trailing block has ||T(k:m, k:n)||_F <= tol ||A||_F."""
        m, n = A.shape
        if not build_uv:
            flags |= RANDUTV_NO_UV
        Tf = colmajor(n, n, device=A.device)
        Uf = colmajor(m, n, device=A.device) if build_uv else None
        V = colmajor(n, n, device=A.device) if build_uv else None
        rho = ctypes.c_double()
        kk = ctypes.c_int64()
        st = self.lib.randutv_factor_tol(self.h, m, n, _ptr(A), _ld(A), float(tol), int(b), int(q),
                                         int(seed) & (2**64 - 1), flags, _ptr(Uf), _ld(Uf) if Uf is not None else 1,
                                         _ptr(Tf), _ld(Tf), _ptr(V), _ld(V) if V is not None else 1,
                                         ctypes.byref(kk), ctypes.byref(rho))
        _check("randutv_factor_tol", st)
        k = kk.value
        return (Uf[:, :k] if Uf is not None else None), Tf[:k, :], V, rho.value, k

    def randutv_hqrrp(self, A, b, seed, build_q=True, flags=0):
        """HQRRP (column-pivoted QR, A P = Q R) of the column-major device matrix A,
        overwritten by R: returns (Q, jpvt) with jpvt an int64 device tensor."""
        import torch
        m, n = A.shape
        if not build_q:
            flags |= RANDUTV_NO_UV
        jpvt = torch.empty(n, dtype=torch.int64, device=A.device)
        Q = colmajor(m, m, device=A.device) if build_q else None
        st = self.lib.randutv_hqrrp(self.h, m, n, _ptr(A), _ld(A), int(b), int(seed) & (2**64 - 1), flags,
                                    _ptr(jpvt), _ptr(Q), _ld(Q) if Q is not None else 1)
        _check("randutv_hqrrp", st)
        return Q, jpvt

    def randutv_hqrrp_rank(self, A, k, b, seed, build_q=True, flags=0):
        """Partial HQRRP (K = ceil(k/b) blocks) of the device matrix A, overwritten by
        R: returns (Q, jpvt, rho) with rho = ||R(k:, k:)||_F."""
        import torch
        m, n = A.shape
        if not build_q:
            flags |= RANDUTV_NO_UV
        jpvt = torch.empty(n, dtype=torch.int64, device=A.device)
        Q = colmajor(m, m, device=A.device) if build_q else None
        rho = ctypes.c_double()
        st = self.lib.randutv_hqrrp_rank(self.h, m, n, _ptr(A), _ld(A), int(k), int(b), int(seed) & (2**64 - 1),
                                         flags, _ptr(jpvt), _ptr(Q), _ld(Q) if Q is not None else 1,
                                         ctypes.byref(rho))
        _check("randutv_hqrrp_rank", st)
        return Q, jpvt, rho.value

    def randutv_hqrrp_host(self, A_host, b, seed):
        """HQRRP_left of the column-major host (numpy, Fortran-order) matrix A_host,
        overwritten by R + Householder tails: returns (jpvt, tau, report)."""
        import numpy as np
        m, n = A_host.shape
        assert A_host.flags.f_contiguous and A_host.dtype == np.float64
        jpvt = np.zeros(n, dtype=np.int64)
        tau = np.zeros(n)
        rep = HostReport()
        st = self.lib.randutv_hqrrp_host(self.h, m, n, A_host.ctypes.data, m, int(b), int(seed) & (2**64 - 1), 0,
                                         jpvt.ctypes.data, tau.ctypes.data, ctypes.byref(rep))
        _check("randutv_hqrrp_host", st)
        return jpvt, tau, {k: getattr(rep, k) for k, _ in HostReport._fields_}

    # ---------------------------------------------------------------- step entries
    def randutv_gaussian(self, seed, it, rows, cols, G=None):
        G = colmajor(rows, cols) if G is None else G
        _check("randutv_gaussian", self.lib.randutv_gaussian(self.h, int(seed) & (2**64 - 1), int(it), rows, cols,
                                                             _ptr(G), max(rows, 1) if G.shape[1] <= 1 else _ld(G)))
        return G

    def randutv_dgemm(self, transa, transb, A, B, C, alpha=1.0, beta=0.0):
        M, N = C.shape
        K = A.shape[0] if transa else A.shape[1]
        _check("randutv_dgemm", self.lib.randutv_dgemm(self.h, int(transa), int(transb), M, N, K, float(alpha),
                                                       _ptr(A), _ld(A), _ptr(B), _ld(B), float(beta), _ptr(C),
                                                       _ld(C)))
        return C

    def randutv_panel_qr(self, P):
        """In-place Householder QR of the column-major panel P: returns (P, tau, Tf)."""
        import torch
        h, w = P.shape
        tau = torch.empty(w, dtype=torch.float64, device=P.device)
        Tf = colmajor(w, w, device=P.device)
        _check("randutv_panel_qr", self.lib.randutv_panel_qr(self.h, h, w, _ptr(P), _ld(P), _ptr(tau), _ptr(Tf),
                                                             _ld(Tf)))
        return P, tau, Tf

    # ---------------------------------------------------------------- host-streamed
    def randutv_factor_host(self, A, b, q, seed, build_uv=True, U=None, V=None, cache_bytes=0, flags=0):
        """Host-streamed randUTV: A (Fortran-ordered float64 numpy array in host memory,
        ideally pinned, see pinned_colmajor) is overwritten by T; returns (U, V, report)."""
        m, n = A.shape
        if not build_uv:
            flags |= RANDUTV_NO_UV
        if build_uv:
            U = pinned_colmajor(m, m) if U is None else U
            V = pinned_colmajor(n, n) if V is None else V
        rep = HostReport()
        st = self.lib.randutv_factor_host(self.h, m, n, _hptr(A), _hld(A), int(b), int(q), int(seed) & (2**64 - 1),
                                          flags, int(cache_bytes), _hptr(U), _hld(U) if U is not None else 1,
                                          _hptr(V), _hld(V) if V is not None else 1, ctypes.byref(rep))
        _check("randutv_factor_host", st)
        return U, V, {k: getattr(rep, k) for k, _ in HostReport._fields_}

    def randutv_factor_host_steps(self, A, U, V, b, q, seed, step_begin, step_end, build_uv=True, cache_bytes=0,
                                  flags=0):
        """Steps [step_begin, step_end) of the host-streamed randUTV on the host state
        (A = T so far, U, V; resumable, see randutv.h); returns the report."""
        m, n = A.shape
        if not build_uv:
            flags |= RANDUTV_NO_UV
        rep = HostReport()
        st = self.lib.randutv_factor_host_steps(self.h, m, n, _hptr(A), _hld(A), int(b), int(q),
                                                int(seed) & (2**64 - 1), flags, int(cache_bytes), _hptr(U),
                                                _hld(U) if U is not None else 1, _hptr(V),
                                                _hld(V) if V is not None else 1, int(step_begin),
                                                min(int(step_end), 2**63 - 1), ctypes.byref(rep))
        _check("randutv_factor_host_steps", st)
        return {k: getattr(rep, k) for k, _ in HostReport._fields_}

    # ---------------------------------------------------------------- multi-GPU
    def comm_init(self, unique_id, nranks, rank):
        """Join the NCCL communicator (collective; one process per GPU)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), RANDUTV_UNIQUE_ID_BYTES)
        _check("randutv_comm_init", self.lib.randutv_comm_init(self.h, buf, int(nranks), int(rank)))

    def comm_init_torch(self, group=None):
        """Bootstrap the communicator over an initialised torch.distributed group:
        rank 0 draws the NCCL unique id, broadcast_object_list ships it."""
        import torch.distributed as dist
        rank, ws = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.comm_init(obj[0], ws, rank)
        return rank, ws

    def randutv_factor_dist(self, A_local, m, n, b, q, seed, build_uv=True, U_local=None, V_local=None, flags=0,
                            nranks=None, rank=None):
        """Sharded randUTV (collective).  A_local (m x n_p, column-major, device) is
        overwritten by this rank's columns of T; returns (U_local, V_local)."""
        import torch.distributed as dist
        if nranks is None:
            nranks, rank = dist.get_world_size(), dist.get_rank()
        lay = dist_layout(m, n, b, nranks, rank)
        if not build_uv:
            flags |= RANDUTV_NO_UV
        if build_uv:
            U_local = colmajor(lay["u1"] - lay["u0"], m, device=A_local.device) if U_local is None else U_local
            V_local = colmajor(lay["v1"] - lay["v0"], n, device=A_local.device) if V_local is None else V_local
        st = self.lib.randutv_factor_dist(self.h, m, n, _ptr(A_local), _ld_or(A_local, m), int(b), int(q),
                                          int(seed) & (2**64 - 1), flags, _ptr(U_local), _ld_or(U_local, 1),
                                          _ptr(V_local), _ld_or(V_local, 1))
        _check("randutv_factor_dist", st)
        return U_local, V_local

    def randutv_factor_dist_rank(self, A_local, m, n, k, b, q, seed, build_uv=True, Uk_local=None, V_local=None,
                                 flags=0, nranks=None, rank=None):
        """Sharded truncated randUTV (collective): returns (Uk_local, V_local, rho)."""
        import torch.distributed as dist
        if nranks is None:
            nranks, rank = dist.get_world_size(), dist.get_rank()
        lay = dist_layout(m, n, b, nranks, rank)
        if not build_uv:
            flags |= RANDUTV_NO_UV
        if build_uv:
            Uk_local = colmajor(lay["u1"] - lay["u0"], k, device=A_local.device) if Uk_local is None else Uk_local
            V_local = colmajor(lay["v1"] - lay["v0"], n, device=A_local.device) if V_local is None else V_local
        rho = ctypes.c_double()
        st = self.lib.randutv_factor_dist_rank(self.h, m, n, _ptr(A_local), _ld_or(A_local, m), int(k), int(b),
                                               int(q), int(seed) & (2**64 - 1), flags, _ptr(Uk_local),
                                               _ld_or(Uk_local, 1), _ptr(V_local), _ld_or(V_local, 1),
                                               ctypes.byref(rho))
        _check("randutv_factor_dist_rank", st)
        return Uk_local, V_local, rho.value

    def randutv_factor_dist_host(self, A_local, m, n, b, q, seed, build_uv=True, U_local=None, V_local=None,
                                 cache_bytes=0, flags=0, nranks=None, rank=None):
        """Sharded + host-streamed randUTV (collective).  A_local (m x n_p,
        Fortran-ordered float64 host array, pinned ideally) is overwritten by this
        rank's columns of T; returns (U_local, V_local, report) in host memory."""
        import torch.distributed as dist
        if nranks is None:
            nranks, rank = dist.get_world_size(), dist.get_rank()
        lay = dist_layout(m, n, b, nranks, rank)
        if not build_uv:
            flags |= RANDUTV_NO_UV
        if build_uv:
            U_local = pinned_colmajor(lay["u1"] - lay["u0"], m) if U_local is None else U_local
            V_local = pinned_colmajor(lay["v1"] - lay["v0"], n) if V_local is None else V_local
        hp = lambda x: x.ctypes.data if x is not None and x.size > 0 else None
        hld = lambda x, d: max(x.strides[1] // 8, 1) if x is not None and x.ndim == 2 and x.size > 0 else d
        rep = HostReport()
        st = self.lib.randutv_factor_dist_host(self.h, m, n, hp(A_local), hld(A_local, m), int(b), int(q),
                                               int(seed) & (2**64 - 1), flags, int(cache_bytes), hp(U_local),
                                               hld(U_local, 1), hp(V_local), hld(V_local, 1), ctypes.byref(rep))
        _check("randutv_factor_dist_host", st)
        return U_local, V_local, rep

    def randutv_small_svd(self, B, allow_nonconvergence=False):
        import torch
        w = B.shape[0]
        Us = colmajor(w, w, device=B.device)
        Vs = colmajor(w, w, device=B.device)
        d = torch.empty(w, dtype=torch.float64, device=B.device)
        st = self.lib.randutv_small_svd(self.h, w, _ptr(B), _ld(B), _ptr(Us), _ptr(d), _ptr(Vs))
        _check("randutv_small_svd", st, allow_positive=allow_nonconvergence)
        return Us, d, Vs, st


def pinned_colmajor(m, n):
    """Fortran-ordered m x n float64 numpy array in pinned (page-locked) host memory."""
    import torch
    return torch.empty((n, m), dtype=torch.float64, pin_memory=True).numpy().T


def _hptr(X):
    if X is None:
        return None
    if not isinstance(X, np.ndarray) or X.dtype != np.float64 or X.strides[0] != 8:
        raise ValueError("host matrices must be column-major float64 numpy arrays")
    return ctypes.c_void_p(X.ctypes.data)


def _hld(X):
    return max(X.strides[1] // 8, X.shape[0], 1) if X.shape[1] > 1 else max(X.shape[0], 1)


def randutv_factor(m, n, A, lda, b, q, seed, U, T, V):
    """The literal north-star entry: all four matrices on the device (torch tensors)
    or all on the host (numpy Fortran-ordered float64 arrays, ideally pinned)."""
    lib = load_library()

    def p(X):
        if isinstance(X, np.ndarray):
            if not X.flags.f_contiguous or X.dtype != np.float64:
                raise ValueError("host arrays must be Fortran-ordered float64")
            return ctypes.c_void_p(X.ctypes.data)
        if hasattr(X, "data_ptr"):
            return ctypes.c_void_p(X.data_ptr())
        return ctypes.c_void_p(int(X))

    st = lib.randutv_factor(int(m), int(n), p(A), int(lda), int(b), int(q), int(seed) & (2**64 - 1),
                            p(U), p(T), p(V))
    _check("randutv_factor", st)
    return st


def randutv_workspace_bytes(m, n, b, q, flags=0):
    lib = load_library()
    out = ctypes.c_size_t()
    _check("randutv_workspace_bytes", lib.randutv_workspace_bytes(m, n, b, q, flags, ctypes.byref(out)))
    return out.value


def randutv_dgemm_plan(M, N, K, ws_elems, sms=148, tail_split=True):
    """The DGEMM work schedule (host arithmetic; include/randutv.h): a dict of the six plan entries."""
    lib = load_library()
    out = (ctypes.c_int64 * 6)()
    _check("randutv_dgemm_plan", lib.randutv_dgemm_plan(int(M), int(N), int(K), int(ws_elems), int(sms),
                                                        int(bool(tail_split)), out))
    return dict(zip(("tiles", "full", "tsplits", "kchunk", "resident", "partial_elems"), (int(v) for v in out)))


# ----------------------------------------------------------------------------- multi-GPU helpers

def dist_layout(m, n, b, nranks, rank):
    """Layout of one rank of the column-sharded path (randutv_dist_layout, host only):
    local column count and the U / V row ranges it holds."""
    lib = load_library()
    out = (_i64 * 5)()
    _check("randutv_dist_layout", lib.randutv_dist_layout(int(m), int(n), int(b), int(nranks), int(rank), out))
    return {"ncols": out[0], "u0": out[1], "u1": out[2], "v0": out[3], "v1": out[4]}


def local_columns(n, b, nranks, rank):
    """Global column indices of a rank's local matrix, in local order (block-cyclic
    by column blocks of width b: global block j on rank j mod nranks)."""
    b = min(int(b), int(n))
    nblocks = (n + b - 1) // b
    cols = []
    for j in range(rank, nblocks, nranks):
        cols.extend(range(j * b, min(n, (j + 1) * b)))
    return np.asarray(cols, dtype=np.int64)


def nccl_unique_id():
    """A fresh NCCL unique id (bytes) for randutv_comm_init."""
    lib = load_library()
    buf = ctypes.create_string_buffer(RANDUTV_UNIQUE_ID_BYTES)
    _check("randutv_nccl_unique_id", lib.randutv_nccl_unique_id(buf))
    return buf.raw


def _ld_or(X, default):
    return _ld(X) if X is not None else max(int(default), 1)


def randutv_factor_dist_loopback(A_locals, m, n, b, q, seed, U_locals=None, V_locals=None, build_uv=True, flags=0,
                                 device=None, k=0):
    """The sharded SPMD driver with len(A_locals) virtual ranks as host threads on one
    GPU (collectives by device copies between host barriers): the single-GPU test
    harness of the multi-GPU path.  A_locals are overwritten with the ranks' T columns."""
    import torch
    lib = load_library()
    P = len(A_locals)
    if device is None:
        device = A_locals[0].device.index if A_locals[0].device.index is not None else torch.cuda.current_device()
    if not build_uv:
        flags |= RANDUTV_NO_UV
    lays = [dist_layout(m, n, b, P, p) for p in range(P)]
    # one leading dimension per matrix kind for all virtual ranks (the row counts differ by one)
    mu = max(l["u1"] - l["u0"] for l in lays)
    nv = max(l["v1"] - l["v0"] for l in lays)
    if build_uv:
        if U_locals is None:
            U_locals = [colmajor(mu, k if k else m, device=f"cuda:{device}")[:l["u1"] - l["u0"]] for l in lays]
        if V_locals is None:
            V_locals = [colmajor(nv, n, device=f"cuda:{device}")[:l["v1"] - l["v0"]] for l in lays]
    lda = max([_ld(a) for a in A_locals if a.numel() > 0] + [m])
    ldu = max(mu, 1)
    ldv = max(nv, 1)
    for X, ld in [(a, lda) for a in A_locals] + ([(u, ldu) for u in U_locals] + [(v, ldv) for v in V_locals]
                                                  if build_uv else []):
        if X.numel() > 0 and X.stride(1) != ld and X.shape[1] > 1:
            raise ValueError("loopback: every rank's matrix of a kind needs the same leading dimension")
    arr = lambda xs: (_vp * P)(*[x.data_ptr() if x is not None and x.numel() > 0 else None for x in xs])
    torch.cuda.synchronize(device)
    rho = ctypes.c_double()
    st = lib.randutv_factor_dist_loopback(int(device), P, int(m), int(n), arr(A_locals), lda, int(b), int(q),
                                          int(seed) & (2**64 - 1), flags, arr(U_locals) if build_uv else None, ldu,
                                          arr(V_locals) if build_uv else None, ldv, int(k), ctypes.byref(rho))
    _check("randutv_factor_dist_loopback", st)
    if k:
        return U_locals, V_locals, rho.value
    return U_locals, V_locals


def randutv_factor_dist_host_loopback(A_locals, m, n, b, q, seed, U_locals=None, V_locals=None, build_uv=True,
                                      flags=0, cache_bytes=0, device=0):
    """The sharded host-streamed driver (randutv_factor_dist_host) with
    len(A_locals) virtual ranks on one GPU.  A_locals: the ranks' block-cyclic
    columns as Fortran-ordered float64 host arrays (pinned ideally), overwritten
    by T; U_locals / V_locals (allocated here if None): the ranks' rows of U, V."""
    lib = load_library()
    P = len(A_locals)
    if not build_uv:
        flags |= RANDUTV_NO_UV
    lays = [dist_layout(m, n, b, P, p) for p in range(P)]
    mu = max(l["u1"] - l["u0"] for l in lays)
    nv = max(l["v1"] - l["v0"] for l in lays)
    if build_uv:
        if U_locals is None:
            U_locals = [pinned_colmajor(mu, m)[:l["u1"] - l["u0"]] for l in lays]
        if V_locals is None:
            V_locals = [pinned_colmajor(nv, n)[:l["v1"] - l["v0"]] for l in lays]
    arr = lambda xs: (_vp * P)(*[x.ctypes.data if x is not None and x.size > 0 else None for x in xs])
    st = lib.randutv_factor_dist_host_loopback(0 if device is None else int(device), P, int(m), int(n), arr(A_locals),
                                               int(m), int(b), int(q), int(seed) & (2**64 - 1), flags,
                                               int(cache_bytes), arr(U_locals) if build_uv else None, max(mu, 1),
                                               arr(V_locals) if build_uv else None, max(nv, 1))
    _check("randutv_factor_dist_host_loopback", st)
    return U_locals, V_locals
