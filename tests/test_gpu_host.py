"""Host-streamed randUTV (the GPU analogue of the
paper's out-of-core cache + overlap runtime) against the CPU
oracle and the in-HBM path.  A tiny device cache (3 panels) forces every pass
to stream, so the serpentine LRU, the write-back ordering, the partial (rows k:m)
panel loads and the fused update/fold/next-sample pass are all exercised; a cache that holds everything must move each
matrix exactly once in and once out."""
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


def _run_host(ctx, A, b, q, seed, cache_panels, pinned=True, build_uv=True):
    from paper_2002_06960_b200.randutv import pinned_colmajor
    m, n = A.shape
    bb = min(b, n)
    Ah = pinned_colmajor(m, n) if pinned else np.zeros((m, n), order="F")
    Ah[:] = A
    slot = max(m, n) * bb * 8
    U, V, rep = ctx.randutv_factor_host(Ah, b, q, seed, cache_bytes=cache_panels * slot, build_uv=build_uv)
    return (np.array(U) if U is not None else None), np.array(Ah), (np.array(V) if V is not None else None), rep


# U, V elementwise bound per case: 1e-11, except (520, 520, 64, 2), whose
# tail singular vectors are ill-conditioned -- the oracle on A vs on
# A(1 + 2^-52 N(0,1)) already differs by 7.2e-12 in |V| (tests/test_parity_calibration.py,
# bounds sit >= 30x above the calibrated noise).
UV_TOL = {(520, 520, 64, 2): 3e-10}


@pytest.mark.parametrize("m,n,b,q", [(300, 300, 32, 1), (400, 250, 40, 2), (129, 129, 128, 0), (64, 40, 64, 1),
                                     (60, 60, 4, 1), (520, 520, 64, 2)])
@pytest.mark.parametrize("cache_panels", [3, 1000])
def test_host_streamed_parity(ctx, m, n, b, q, cache_panels):
    uv_tol = UV_TOL.get((m, n, b, q), ELEM_TOL)
    rng = np.random.default_rng(3 * m + n + b)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    U, T, V, rep = _run_host(ctx, A, b, q, 41, cache_panels)
    o = oracle_randutv(A, b, q, 41)
    nA = np.linalg.norm(A)
    assert recon_error(A, U, T, V) <= 1e-12
    assert spectral_orth_error(U) <= 1e-12 and spectral_orth_error(V) <= 1e-12
    assert np.all(np.tril(T, -1) == 0.0)
    assert diag_parity(np.diag(T), np.diag(o["T"])) <= 1.0
    assert np.max(np.abs(np.abs(T) - np.abs(o["T"]))) / nA <= ELEM_TOL
    assert np.max(np.abs(np.abs(U) - np.abs(o["U"]))) <= uv_tol
    assert np.max(np.abs(np.abs(V) - np.abs(o["V"]))) <= uv_tol
    Ug, Tg, Vg, _ = ctx.randutv_factor_ex(to_dev(A), b, q, 41)
    assert np.max(np.abs(np.abs(T) - np.abs(to_np(Tg)))) / nA <= ELEM_TOL
    if cache_panels >= 1000:
        # everything resident: A in once, T, U, V out once
        assert rep["h2d_bytes"] == 8 * m * n
        assert rep["d2h_bytes"] == 8 * (m * n + m * m + n * n)
    else:
        assert rep["cache_slots"] == 3 and rep["h2d_bytes"] > 8 * m * n


def test_host_streamed_unpinned_and_no_uv(ctx):
    rng = np.random.default_rng(17)
    A = np.asfortranarray(rng.standard_normal((256, 200)))
    _, T1, _, _ = _run_host(ctx, A, 32, 1, 5, 4, pinned=False, build_uv=False)
    _, T2, _, rep = _run_host(ctx, A, 32, 1, 5, 4, pinned=True, build_uv=True)
    assert np.array_equal(T1, T2)
    assert rep["wall_ms"] > 0 and rep["h2d_ms"] > 0


def test_host_streamed_nonfinite(ctx):
    from paper_2002_06960_b200.randutv import RANDUTV_CHECK_FINITE, RANDUTV_ERR_NONFINITE, RandUTVError
    A = np.ones((64, 64), order="F")
    A[10, 50] = np.inf
    with pytest.raises(RandUTVError) as e:
        ctx.randutv_factor_host(A, 16, 1, 1, build_uv=False, flags=RANDUTV_CHECK_FINITE, cache_bytes=3 * 64 * 16 * 8)
    assert e.value.status == RANDUTV_ERR_NONFINITE


@pytest.mark.parametrize("cuts", [[2], [1, 3, 5], [7]])
def test_host_streamed_resume(ctx, cuts):
    """randutv_factor_host_steps (resumable per iteration):
    the host state (j, T, U, V) after steps [0, j) is a complete checkpoint --
    a fresh context resumes from copies of it, and the ranges give the single
    call's factorisation (and the oracle's) to rounding."""
    from paper_2002_06960_b200.randutv import Context, pinned_colmajor
    m, n, b, q, seed = 300, 280, 32, 1, 17   # 8 sampled steps + a final block
    rng = np.random.default_rng(99)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    U1, T1, V1, _ = _run_host(ctx, A, b, q, seed, 4)
    Ah, Uh, Vh = pinned_colmajor(m, n), pinned_colmajor(m, m), pinned_colmajor(n, n)
    Ah[:] = A
    bounds = [0] + cuts + [2 ** 62]
    for lo, hi in zip(bounds, bounds[1:]):
        c = Context()   # a new process / context per range: only the host state carries over
        try:
            ck = (np.array(Ah), np.array(Uh), np.array(Vh))   # the checkpoint, restored below
            Ah[:], Uh[:], Vh[:] = ck
            c.randutv_factor_host_steps(Ah, Uh, Vh, b, q, seed, lo, hi, cache_bytes=4 * max(m, n) * b * 8)
        finally:
            c.close()
    T2, U2, V2 = np.array(Ah), np.array(Uh), np.array(Vh)
    nA = np.linalg.norm(A)
    assert np.max(np.abs(T2 - T1)) / nA <= 1e-13
    assert np.max(np.abs(U2 - U1)) <= 1e-12 and np.max(np.abs(V2 - V1)) <= 1e-12
    o = oracle_randutv(A, b, q, seed)
    assert recon_error(A, U2, T2, V2) <= 1e-12
    assert diag_parity(np.diag(T2), np.diag(o["T"])) <= 1.0
    assert np.max(np.abs(np.abs(T2) - np.abs(o["T"]))) / nA <= ELEM_TOL


def test_host_streamed_resume_t_only_belady(ctx):
    """T-only ranges (the Belady plan is rebuilt per range from its first step)
    give the single call's T to rounding."""
    from paper_2002_06960_b200.randutv import pinned_colmajor
    m, n, b, q, seed = 400, 400, 32, 2, 23
    A = np.asfortranarray(np.random.default_rng(5).standard_normal((m, n)))
    _, T1, _, _ = _run_host(ctx, A, b, q, seed, 5, build_uv=False)
    Ah = pinned_colmajor(m, n)
    Ah[:] = A
    for lo, hi in [(0, 4), (4, 9), (9, 2 ** 62)]:
        ctx.randutv_factor_host_steps(Ah, None, None, b, q, seed, lo, hi, build_uv=False,
                                      cache_bytes=5 * max(m, n) * b * 8)
    assert np.max(np.abs(np.array(Ah) - T1)) / np.linalg.norm(A) <= 1e-13


def test_host_streamed_resume_arguments(ctx):
    from paper_2002_06960_b200.randutv import RandUTVError
    A = np.zeros((64, 64), order="F")
    with pytest.raises(RandUTVError) as e:
        ctx.randutv_factor_host_steps(A, None, None, 16, 1, 1, 3, 3, build_uv=False)
    assert e.value.status == -16
    with pytest.raises(RandUTVError) as e:
        ctx.randutv_factor_host_steps(A, None, None, 16, 1, 1, 9, 12, build_uv=False)
    assert e.value.status == -15


@pytest.mark.parametrize("m,n,b,q,slots", [(2048, 2048, 128, 1, 5), (3000, 2500, 128, 2, 8), (4096, 4096, 128, 1, 12)])
def test_host_streamed_traffic_model(ctx, m, n, b, q, slots):
    """a T-only host-streamed run moves the PCIe bytes of the
    replay model paper_2002_06960_b200.flops.host_stream_traffic under Belady
    eviction (within the prefetch's slack: measured 0.3-4 %), and fewer than
    LRU would on the same access sequence."""
    from paper_2002_06960_b200.flops import host_stream_traffic
    from paper_2002_06960_b200.randutv import pinned_colmajor
    A = pinned_colmajor(m, n)
    A[:] = np.random.default_rng(m + n).standard_normal((m, n))
    slot = ((max(m, n) * b + 31) // 32) * 32 * 8
    _, _, rep = ctx.randutv_factor_host(A, b, q, 3, build_uv=False, cache_bytes=slots * slot)
    hb, db = host_stream_traffic(m, n, b, q, rep["cache_slots"], "belady")
    hl, dl = host_stream_traffic(m, n, b, q, rep["cache_slots"], "lru")
    assert hb <= rep["h2d_bytes"] <= 1.05 * hb and db <= rep["d2h_bytes"] <= 1.06 * db
    assert rep["h2d_bytes"] < hl


def _shard_host_run(A, b, q, seed, P, cache_panels, build_uv=True):
    """randutv_factor_dist_host (sharded + host-streamed, SURVEY.md §8(f)
    NEXT-1) with P loopback ranks: every rank's block-cyclic columns and U/V
    rows live in pinned host memory and stream through a cache_panels-slot
    device cache per rank."""
    from paper_2002_06960_b200.randutv import (dist_layout, local_columns, pinned_colmajor,
                                               randutv_factor_dist_host_loopback)
    m, n = A.shape
    bb = min(b, n)
    locals_ = []
    for p in range(P):
        cols = local_columns(n, b, P, p)
        Al = pinned_colmajor(m, max(len(cols), 1))[:, :len(cols)]
        Al[:] = A[:, cols]
        locals_.append(Al)
    slot = max(m, n) * bb * 8
    Us, Vs = randutv_factor_dist_host_loopback(locals_, m, n, b, q, seed, build_uv=build_uv,
                                               cache_bytes=cache_panels * slot)
    T = np.zeros((m, n), order="F")
    for p in range(P):
        cols = local_columns(n, b, P, p)
        if len(cols):
            T[:, cols] = locals_[p]
    if not build_uv:
        return None, T, None
    U = np.zeros((m, m), order="F")
    V = np.zeros((n, n), order="F")
    for p in range(P):
        lay = dist_layout(m, n, b, P, p)
        if lay["u1"] > lay["u0"]:
            U[lay["u0"]:lay["u1"], :] = Us[p]
        if lay["v1"] > lay["v0"]:
            V[lay["v0"]:lay["v1"], :] = Vs[p]
    return U, T, V


@pytest.mark.parametrize("m,n,b,q,P", [
    (300, 300, 32, 1, 2),
    (400, 250, 40, 2, 3),     # tall, ragged, 3 ranks
    (96, 96, 32, 1, 4),       # a rank with no column
    (129, 129, 128, 0, 2),    # final block of one column
    (64, 40, 64, 1, 3),       # b >= n: QR + SVD only
])
@pytest.mark.parametrize("cache_panels", [3, 1000])
def test_dist_host_parity(ctx, m, n, b, q, P, cache_panels):
    rng = np.random.default_rng(5 * m + n + b + 11 * P)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    U, T, V = _shard_host_run(A, b, q, 23, P, cache_panels)
    o = oracle_randutv(A, b, q, 23)
    nA = np.linalg.norm(A)
    assert recon_error(A, U, T, V) <= 1e-12
    assert spectral_orth_error(U) <= 1e-12 and spectral_orth_error(V) <= 1e-12
    assert np.all(np.tril(T, -1) == 0.0)
    assert diag_parity(np.diag(T), np.diag(o["T"])) <= 1.0
    assert np.max(np.abs(np.abs(T) - np.abs(o["T"]))) / nA <= ELEM_TOL
    assert np.max(np.abs(np.abs(U) - np.abs(o["U"]))) <= ELEM_TOL
    assert np.max(np.abs(np.abs(V) - np.abs(o["V"]))) <= ELEM_TOL


def test_dist_host_matches_dist_and_no_uv(ctx):
    """Same layout, same collectives: the host-streamed sharded T equals the
    in-HBM sharded T to rounding, is deterministic, and does not depend on U, V."""
    import torch
    from paper_2002_06960_b200.randutv import colmajor, local_columns, randutv_factor_dist_loopback
    rng = np.random.default_rng(77)
    m, n, b, q, P = 360, 300, 32, 1, 3
    A = np.asfortranarray(rng.standard_normal((m, n)))
    r1 = _shard_host_run(A, b, q, 5, P, 3)
    r2 = _shard_host_run(A, b, q, 5, P, 3)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)
    _, T3, _ = _shard_host_run(A, b, q, 5, P, 3, build_uv=False)
    assert np.array_equal(T3, r1[1])
    locs = []
    for p in range(P):
        cols = local_columns(n, b, P, p)
        Al = colmajor(m, len(cols))
        Al.copy_(torch.from_numpy(np.ascontiguousarray(A[:, cols])))
        locs.append(Al)
    randutv_factor_dist_loopback(locs, m, n, b, q, 5, build_uv=False)
    Td = np.zeros((m, n), order="F")
    for p in range(P):
        Td[:, local_columns(n, b, P, p)] = to_np(locs[p])
    assert np.max(np.abs(np.abs(Td) - np.abs(r1[1]))) / np.linalg.norm(A) <= ELEM_TOL
