"""The column-sharded multi-GPU randUTV on one GPU.

`randutv_factor_dist_loopback` runs the SAME SPMD driver as
`randutv_factor_dist` (NCCL, one process per GPU) with P virtual ranks as host
threads; only the four collectives differ (device copies / fixed-order sums
between host barriers instead of NCCL).  The assembled U, T, V are checked
against the CPU oracle with the north-star tolerances, exactly like the
single-GPU path (tests/test_gpu_randutv.py), and against the single-GPU result.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import diag_parity, recon_error, spectral_orth_error, to_dev, to_np  # noqa: E402
from oracle.randutv import randutv as oracle_randutv  # noqa: E402

ELEM_TOL = 1e-11


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    from paper_2002_06960_b200.randutv import Context
    c = Context()
    yield c
    c.close()


def shard_and_run(A, b, q, seed, P, build_uv=True):
    import torch
    from paper_2002_06960_b200.randutv import (colmajor, dist_layout, local_columns,
                                               randutv_factor_dist_loopback)
    m, n = A.shape
    locals_ = []
    for p in range(P):
        cols = local_columns(n, b, P, p)
        Al = colmajor(m, len(cols))
        if len(cols):
            Al.copy_(torch.from_numpy(np.ascontiguousarray(A[:, cols])))
        locals_.append(Al)
    Us, Vs = randutv_factor_dist_loopback(locals_, m, n, b, q, seed, build_uv=build_uv)
    T = np.zeros((m, n), order="F")
    for p in range(P):
        cols = local_columns(n, b, P, p)
        if len(cols):
            T[:, cols] = to_np(locals_[p])
    if not build_uv:
        return None, T, None
    U = np.zeros((m, m), order="F")
    V = np.zeros((n, n), order="F")
    for p in range(P):
        lay = dist_layout(m, n, b, P, p)
        if lay["u1"] > lay["u0"]:
            U[lay["u0"]:lay["u1"], :] = to_np(Us[p])
        if lay["v1"] > lay["v0"]:
            V[lay["v0"]:lay["v1"], :] = to_np(Vs[p])
    return U, T, V


@pytest.mark.parametrize("m,n,b,q,P", [
    (256, 256, 32, 1, 2),
    (300, 300, 32, 2, 3),      # ragged final block, 3 ranks
    (400, 250, 40, 1, 2),      # tall, ragged
    (200, 200, 64, 1, 4),      # 4 blocks on 4 ranks (last ragged)
    (96, 96, 32, 1, 4),        # fewer blocks than ranks: rank 3 holds no column
    (129, 129, 128, 0, 2),     # final block of one column
    (64, 40, 64, 1, 3),        # b >= n: QR + SVD only, owner 0
    (520, 520, 64, 2, 8),      # 8 ranks
])
def test_dist_loopback_parity(ctx, m, n, b, q, P):
    rng = np.random.default_rng(7 * m + n + b + 13 * P)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    U, T, V = shard_and_run(A, b, q, 31, P)
    o = oracle_randutv(A, b, q, 31)
    nA = np.linalg.norm(A)
    assert recon_error(A, U, T, V) <= 1e-12
    assert spectral_orth_error(U) <= 1e-12
    assert spectral_orth_error(V) <= 1e-12
    assert np.all(np.tril(T, -1) == 0.0)
    assert diag_parity(np.diag(T), np.diag(o["T"])) <= 1.0
    assert np.max(np.abs(np.abs(T) - np.abs(o["T"]))) / nA <= ELEM_TOL
    assert np.max(np.abs(np.abs(U) - np.abs(o["U"]))) <= ELEM_TOL
    assert np.max(np.abs(np.abs(V) - np.abs(o["V"]))) <= ELEM_TOL
    # against the single-GPU path on the same A
    Ug, Tg, Vg, _ = ctx.randutv_factor_ex(to_dev(A), b, q, 31)
    assert np.max(np.abs(np.abs(T) - np.abs(to_np(Tg)))) / nA <= ELEM_TOL


def test_dist_loopback_c2_shape(ctx):
    # c2's proportions (Gaussian, b=128, q=1) at n = 1024 on 4 ranks
    from paper_2002_06960_b200.inputs import make_numpy
    A = make_numpy("gauss", 1024, 1024, cfg_index=2)
    U, T, V = shard_and_run(A, 128, 1, 2002, 4)
    o = oracle_randutv(A, 128, 1, 2002)
    assert recon_error(A, U, T, V) <= 1e-12
    assert spectral_orth_error(U) <= 1e-12 and spectral_orth_error(V) <= 1e-12
    assert diag_parity(np.diag(T), np.diag(o["T"])) <= 1.0
    assert np.max(np.abs(np.abs(T) - np.abs(o["T"]))) / np.linalg.norm(A) <= ELEM_TOL


def test_dist_loopback_deterministic_and_no_uv(ctx):
    rng = np.random.default_rng(5)
    A = np.asfortranarray(rng.standard_normal((300, 260)))
    r1 = shard_and_run(A, 32, 1, 9, 3)
    r2 = shard_and_run(A, 32, 1, 9, 3)
    for a, b in zip(r1, r2):
        assert np.array_equal(a, b)
    _, T3, _ = shard_and_run(A, 32, 1, 9, 3, build_uv=False)
    assert np.array_equal(T3, r1[1])   # T does not depend on U, V


def test_dist_requires_comm(ctx):
    import ctypes
    from paper_2002_06960_b200.randutv import RANDUTV_ERR_NOCOMM, colmajor
    A = colmajor(8, 8)
    st = ctx.lib.randutv_factor_dist(ctx.h, 8, 8, ctypes.c_void_p(A.data_ptr()), 8, 4, 1, 1, 1, None, 1, None, 1)
    assert st == RANDUTV_ERR_NOCOMM


@pytest.mark.parametrize("m,n,k,b,q,P", [
    (400, 300, 64, 32, 1, 2),     # k = 2b
    (600, 240, 100, 40, 2, 3),    # k not a multiple of b, ragged rows over 3 ranks
    (4096, 1024, 256, 64, 2, 4),  # c4's proportions at 1/64 of the size (as test_truncated_tall_parity)
])
def test_dist_loopback_truncated(ctx, m, n, k, b, q, P):
    import torch
    from paper_2002_06960_b200.inputs import make_numpy
    from paper_2002_06960_b200.randutv import colmajor, dist_layout, local_columns, randutv_factor_dist_loopback
    if m == 4096:
        A = make_numpy("lowrank", m, n, cfg_index=4, rank=200)
    else:
        A = np.asfortranarray(np.random.default_rng(m + n + k).standard_normal((m, n)))
    locals_ = []
    for p in range(P):
        cols = local_columns(n, b, P, p)
        Al = colmajor(m, len(cols))
        Al.copy_(torch.from_numpy(np.ascontiguousarray(A[:, cols])))
        locals_.append(Al)
    Us, Vs, rho = randutv_factor_dist_loopback(locals_, m, n, b, q, 77, k=k)
    T = np.zeros((m, n), order="F")
    Uk = np.zeros((m, k), order="F")
    V = np.zeros((n, n), order="F")
    for p in range(P):
        cols = local_columns(n, b, P, p)
        T[:, cols] = to_np(locals_[p])
        lay = dist_layout(m, n, b, P, p)
        Uk[lay["u0"]:lay["u1"], :] = to_np(Us[p])
        V[lay["v0"]:lay["v1"], :] = to_np(Vs[p])
    Tk = T[:k, :]
    o = oracle_randutv(A, b, q, 77, k=k, thin_u=True)
    nA = np.linalg.norm(A)
    assert abs(rho - o["rho"]) <= 1e-9 * o["rho"]
    assert diag_parity(np.diag(Tk), np.diag(o["Tk"])) <= 1.0
    assert np.max(np.abs(np.abs(Tk) - np.abs(o["Tk"]))) / nA <= ELEM_TOL
    assert np.max(np.abs(np.abs(Uk) - np.abs(o["Uk"]))) <= 1e-9
    assert spectral_orth_error(Uk) <= 1e-12 and spectral_orth_error(V) <= 1e-12
    assert abs(np.linalg.norm(A - Uk @ Tk @ V.T) - rho) <= 1e-12 * nA


def test_nccl_single_rank_end_to_end(ctx):
    """The NCCL back end itself (dlopen of torch's libnccl.so.2, ncclCommInitRank,
    ncclCommSplit for the side communicator, AllReduce / AllGather / Broadcast /
    AllReduce-min on the ctx streams) through randutv_factor_dist with one rank --
    the only NCCL configuration a single GPU can run without co-scheduled ranks
    waiting on each other."""
    import torch
    from paper_2002_06960_b200.randutv import Context, colmajor, nccl_unique_id
    rng = np.random.default_rng(21)
    m, n, b, q = 300, 260, 32, 1
    A = np.asfortranarray(rng.standard_normal((m, n)))
    c = Context()
    try:
        c.comm_init(nccl_unique_id(), 1, 0)
        Ad = to_dev(A).clone(memory_format=torch.contiguous_format)
        Al = colmajor(m, n)
        Al.copy_(torch.from_numpy(np.ascontiguousarray(A)))
        U, V = c.randutv_factor_dist(Al, m, n, b, q, 17, nranks=1, rank=0)
        torch.cuda.synchronize()
        T = to_np(Al)
        U, V = to_np(U), to_np(V)
        o = oracle_randutv(A, b, q, 17)
        assert recon_error(A, U, T, V) <= 1e-12
        assert spectral_orth_error(U) <= 1e-12 and spectral_orth_error(V) <= 1e-12
        assert diag_parity(np.diag(T), np.diag(o["T"])) <= 1.0
        assert np.max(np.abs(np.abs(T) - np.abs(o["T"]))) / np.linalg.norm(A) <= ELEM_TOL
        # truncated sharded entry on the same communicator
        Al.copy_(torch.from_numpy(np.ascontiguousarray(A)))
        Uk, Vk, rho = c.randutv_factor_dist_rank(Al, m, n, 64, b, q, 17, nranks=1, rank=0)
        to = oracle_randutv(A, b, q, 17, k=64, thin_u=True)
        assert abs(rho - to["rho"]) <= 1e-9 * to["rho"]
        assert np.max(np.abs(np.abs(to_np(Uk)) - np.abs(to["Uk"]))) <= 1e-9
        # sharded + host-streamed entry (NEXT-1) on the same communicator, 3-panel cache
        from paper_2002_06960_b200.randutv import pinned_colmajor
        Ah = pinned_colmajor(m, n)
        Ah[:] = A
        Uh, Vh, rep = c.randutv_factor_dist_host(Ah, m, n, b, q, 17, cache_bytes=3 * m * b * 8, nranks=1, rank=0)
        assert rep.h2d_bytes > 0 and rep.cache_slots == 3
        assert recon_error(A, Uh, Ah, Vh) <= 1e-12
        assert np.max(np.abs(np.abs(Ah) - np.abs(o["T"]))) / np.linalg.norm(A) <= ELEM_TOL
    finally:
        c.close()


def test_nccl_async_graph_capture():
    """RANDUTV_ASYNC on the sharded NCCL path: no host synchronisation inside the
    call (the pre-collective agreement is skipped, the status AllReduce is
    enqueued), so after a warm-up call the whole sharded factorisation -- NCCL
    collectives, V/U stream and comm stream forks included -- is captured into a
    CUDA graph; replays give the eager call's bits; randutv_wait returns the
    status through the communicator.  The loopback communicator (host barriers)
    rejects the flag."""
    import ctypes
    import torch
    from paper_2002_06960_b200.randutv import RANDUTV_ASYNC, Context, colmajor, nccl_unique_id
    rng = np.random.default_rng(22)
    m, n, b, q = 320, 256, 32, 1
    A = np.asfortranarray(rng.standard_normal((m, n)))
    s = torch.cuda.Stream()
    c = Context(0, s)
    try:
        c.comm_init(nccl_unique_id(), 1, 0)
        A0 = colmajor(m, n)
        A0.copy_(torch.from_numpy(np.ascontiguousarray(A)))
        Al = colmajor(m, n)
        U, V = colmajor(m, m), colmajor(n, n)
        Al.copy_(A0)
        c.randutv_factor_dist(Al, m, n, b, q, 5, U_local=U, V_local=V, nranks=1, rank=0)
        T_ref, U_ref, V_ref = Al.clone(), U.clone(), V.clone()
        Al.copy_(A0)
        with torch.cuda.stream(s):
            c.randutv_factor_dist(Al, m, n, b, q, 5, U_local=U, V_local=V, nranks=1, rank=0, flags=RANDUTV_ASYNC)
        assert c.wait() == 0
        assert torch.equal(Al, T_ref) and torch.equal(U, U_ref) and torch.equal(V, V_ref)
        g = torch.cuda.CUDAGraph()
        Al.copy_(A0)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            c.randutv_factor_dist(Al, m, n, b, q, 5, U_local=U, V_local=V, nranks=1, rank=0, flags=RANDUTV_ASYNC)
        for rep in range(2):
            Al.copy_(A0)
            U.zero_()
            V.zero_()
            torch.cuda.synchronize()
            g.replay()
            assert c.wait() == 0
            assert torch.equal(Al, T_ref) and torch.equal(U, U_ref) and torch.equal(V, V_ref)
    finally:
        c.close()
    # the loopback back end cannot be captured: -9
    from paper_2002_06960_b200.randutv import randutv_factor_dist_loopback, RandUTVError
    Als = [to_dev(A[:, :n // 2]), to_dev(A[:, n // 2:])]
    with pytest.raises(RandUTVError) as e:
        randutv_factor_dist_loopback(Als, m, n, n // 2, q, 5, flags=RANDUTV_ASYNC)
    assert e.value.status == -9
