"""HQRRP on the GPU (csrc/hqrrp.cu, through the C ABI `randutv_hqrrp`) against
the CPU oracle (oracle/hqrrp.py).

The pivots are integer decisions taken in FP64 on both sides: jpvt must be
identical.  R and Q are compared elementwise (same dlarfg sign convention on
both sides, so no sign freedom) and through the invariants A P = Q R,
Q^T Q = I, R upper trapezoidal with exact zeros."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import spectral_orth_error, to_dev, to_np  # noqa: E402
from oracle.hqrrp import hqrrp as oracle_hqrrp  # noqa: E402

ELEM_TOL = 1e-11


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    from paper_2002_06960_b200.randutv import Context
    c = Context()
    yield c
    c.close()


def _gpu(ctx, A, b, seed, build_q=True):
    Ad = to_dev(A)
    Q, jp = ctx.randutv_hqrrp(Ad, b, seed, build_q=build_q)
    return (to_np(Q) if Q is not None else None), to_np(Ad), jp.cpu().numpy()


@pytest.mark.parametrize("m,n,b", [
    (300, 200, 32),     # tall, ragged last block
    (200, 200, 64),     # ragged
    (129, 129, 128),    # last block of one column
    (64, 40, 64),       # b >= n: one block
    (50, 50, 1),        # b = 1
    (257, 100, 24),
    (520, 520, 64),     # sketch with 64 rows (RPL 2), 9 blocks
    (1000, 300, 100),   # rows not a multiple of 32 in the sketch
    (700, 600, 300),    # RPL 16 path (b = 300 -> 10 rows per lane)
])
def test_hqrrp_parity(ctx, m, n, b):
    A = np.asfortranarray(np.random.default_rng(m + 7 * n + b).standard_normal((m, n)))
    Q, R, jp = _gpu(ctx, A, b, 77)
    Qo, Ro, jpo = oracle_hqrrp(A, b, 77)
    nA = np.linalg.norm(A)
    assert np.array_equal(jp, jpo)
    assert np.all(np.tril(R, -1) == 0.0)
    assert np.linalg.norm(A[:, jp] - Q @ R) <= 1e-12 * nA
    assert spectral_orth_error(Q) <= 1e-12
    assert np.max(np.abs(R - Ro)) / nA <= ELEM_TOL
    assert np.max(np.abs(Q - Qo)) <= ELEM_TOL
    # R without Q is the same computation
    _, R2, jp2 = _gpu(ctx, A, b, 77, build_q=False)
    assert np.array_equal(jp2, jp) and np.array_equal(R2, R)


def test_hqrrp_rank_revealing_and_deterministic(ctx):
    rng = np.random.default_rng(12)
    m, n, rank, b = 600, 400, 150, 32
    A = np.asfortranarray(rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)))
    Q, R, jp = _gpu(ctx, A, b, 3)
    _, Ro, jpo = oracle_hqrrp(A, b, 3, build_q=False)
    nA = np.linalg.norm(A)
    assert np.array_equal(jp[:rank], jpo[:rank])          # beyond the rank: noise-level pivots
    assert np.linalg.norm(R[rank:, rank:]) <= 1e-12 * nA
    assert np.linalg.norm(A[:, jp] - Q @ R) <= 1e-12 * nA
    Q2, R2, jp2 = _gpu(ctx, A, b, 3)
    assert np.array_equal(jp2, jp) and np.array_equal(R2, R) and np.array_equal(Q2, Q)


def test_hqrrp_orthogonal_columns_sorted(ctx):
    # columns q_c sigma_c with sigma 10^-1.5 apart: pivots in decreasing sigma
    rng = np.random.default_rng(3)
    m, n, b = 256, 10, 4
    Q0, _ = np.linalg.qr(rng.standard_normal((m, n)))
    sig = 10.0 ** (-1.5 * np.arange(n))
    order = rng.permutation(n)
    A = np.asfortranarray(Q0 * sig[order])
    _, R, jp = _gpu(ctx, A, b, 5, build_q=False)
    assert np.array_equal(order[jp], np.arange(n))
    assert np.allclose(np.abs(np.diag(R)), sig, rtol=1e-12, atol=0)


def test_hqrrp_larger_against_oracle(ctx):
    """2048^2, b = 128 (16 blocks, the sketch CPQR at 128 x 2048): pivots exact."""
    A = np.asfortranarray(np.random.default_rng(2048).standard_normal((2048, 2048)))
    Q, R, jp = _gpu(ctx, A, 128, 9)
    _, Ro, jpo = oracle_hqrrp(A, 128, 9, build_q=False)
    nA = np.linalg.norm(A)
    assert np.array_equal(jp, jpo)
    assert np.max(np.abs(R - Ro)) / nA <= ELEM_TOL
    x = np.random.default_rng(1).standard_normal(2048)
    assert np.linalg.norm(A[:, jp] @ x - Q @ (R @ x)) <= 1e-12 * nA * np.linalg.norm(x)


def test_hqrrp_errors(ctx):
    import torch
    from paper_2002_06960_b200.randutv import RandUTVError, colmajor
    A = colmajor(600, 600)
    with pytest.raises(RandUTVError) as e:
        ctx.randutv_hqrrp(A, 600, 1)                       # min(b, n) > 512
    assert e.value.status == -6
    A = colmajor(10, 20)
    with pytest.raises(RandUTVError) as e:
        ctx.randutv_hqrrp(A, 4, 1)                         # m < n
    assert e.value.status == -2
    st = ctx.lib.randutv_hqrrp(ctx.h, 10, 10, None, 10, 4, 1, 0, None, None, 10)
    assert st == -4
    torch.cuda.synchronize()


@pytest.mark.parametrize("m,n,b", [(300, 200, 32), (200, 200, 64), (129, 129, 128), (64, 40, 64), (257, 100, 24),
                                   (520, 520, 64), (1000, 300, 100)])
def test_hqrrp_host_left_parity(ctx, m, n, b):
    """HQRRP_left from host memory against the right-looking oracle:
    same pivots, same R, and the stored Householder tails + tau form the
    oracle's Q (LAPACK dorgqr)."""
    import scipy.linalg.lapack as lp
    from paper_2002_06960_b200.randutv import pinned_colmajor
    A = np.asfortranarray(np.random.default_rng(m + 7 * n + b).standard_normal((m, n)))
    Ah = pinned_colmajor(m, n)
    Ah[:] = A
    jp, tau, rep = ctx.randutv_hqrrp_host(Ah, b, 77)
    Qo, Ro, jpo = oracle_hqrrp(A, b, 77)
    nA = np.linalg.norm(A)
    assert np.array_equal(jp, jpo)
    R = np.triu(Ah)
    assert np.max(np.abs(R - Ro)) / nA <= ELEM_TOL
    Q, _, info = lp.dorgqr(np.array(Ah, order="F"), tau)
    assert info == 0
    assert np.max(np.abs(Q - Qo[:, :n])) <= ELEM_TOL
    assert np.linalg.norm(A[:, jp] - Q @ R[:n, :]) <= 1e-12 * nA
    # left-looking: the host matrix is written once per block plus the moved columns
    assert rep["d2h_bytes"] <= 8 * m * n + 8 * n + 8 * m * 2 * b * (-(-n // b))
    assert rep["h2d_bytes"] >= 8 * m * n


def test_hqrrp_host_unpinned_and_errors(ctx):
    from paper_2002_06960_b200.randutv import RandUTVError
    A = np.asfortranarray(np.random.default_rng(5).standard_normal((150, 90)))
    Ah = A.copy(order="F")                   # pageable: registered for the call
    jp, tau, _ = ctx.randutv_hqrrp_host(Ah, 16, 3)
    _, Ro, jpo = oracle_hqrrp(A, 16, 3, build_q=False)
    assert np.array_equal(jp, jpo)
    assert np.max(np.abs(np.triu(Ah) - Ro)) <= 1e-11 * np.linalg.norm(A)
    with pytest.raises(RandUTVError) as e:
        ctx.randutv_hqrrp_host(np.zeros((10, 20), order="F"), 4, 1)
    assert e.value.status == -2


@pytest.mark.parametrize("m,n,k,b", [(300, 200, 64, 32), (300, 200, 50, 32), (520, 520, 200, 64), (129, 129, 129, 128)])
def test_hqrrp_partial_parity(ctx, m, n, k, b):
    A = np.asfortranarray(np.random.default_rng(m + n + k).standard_normal((m, n)))
    Ad = to_dev(A)
    Q, jp, rho = ctx.randutv_hqrrp_rank(Ad, k, b, 13)
    Q, R, jp = to_np(Q), to_np(Ad), jp.cpu().numpy()
    Qo, Ro, jpo, rho_o = oracle_hqrrp(A, b, 13, k=k)
    nA = np.linalg.norm(A)
    assert np.array_equal(jp, jpo)
    assert abs(rho - rho_o) <= 1e-9 * rho_o + 1e-14 * nA
    assert np.max(np.abs(R - Ro)) / nA <= ELEM_TOL
    assert np.max(np.abs(Q - Qo)) <= ELEM_TOL
    assert np.linalg.norm(A[:, jp] - Q @ R) <= 1e-12 * nA


@pytest.mark.parametrize("m,n,b", [(1, 1, 1), (5, 1, 4), (7, 3, 1), (33, 33, 33), (40, 2, 64)])
def test_hqrrp_degenerate_shapes(ctx, m, n, b):
    """Single column / single row / b = 1 / b > n: in-HBM, partial and host-streamed entries."""
    from paper_2002_06960_b200.randutv import pinned_colmajor
    A = np.asfortranarray(np.random.default_rng(m * 31 + n).standard_normal((m, n)))
    Q, R, jp = _gpu(ctx, A, b, 4)
    Qo, Ro, jpo = oracle_hqrrp(A, b, 4)
    nA = np.linalg.norm(A)
    assert np.array_equal(jp, jpo)
    assert np.max(np.abs(R - Ro)) <= 1e-12 * nA and np.max(np.abs(Q - Qo)) <= 1e-12
    Ad = to_dev(A)
    _, jpk, rho = ctx.randutv_hqrrp_rank(Ad, 1, b, 4, build_q=False)
    _, _, jpko, rho_o = oracle_hqrrp(A, b, 4, build_q=False, k=1)
    assert np.array_equal(jpk.cpu().numpy(), jpko) and abs(rho - rho_o) <= 1e-12 * nA
    Ah = pinned_colmajor(m, n)
    Ah[:] = A
    jph, tau, _ = ctx.randutv_hqrrp_host(Ah, b, 4)
    assert np.array_equal(jph, jpo)
    assert np.max(np.abs(np.triu(Ah) - Ro)) <= 1e-12 * nA
