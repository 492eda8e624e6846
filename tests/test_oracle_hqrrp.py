"""Pins of the HQRRP oracle (oracle/hqrrp.py)
against things other than itself: LAPACK's dgeqp3 (scipy) for the sketch
CPQR, the factorisation invariants A P = Q R, exact column-norm ordering for a
matrix with orthogonal, geometrically scaled columns, and exact rank
revelation on a rank-deficient matrix."""
import numpy as np
import pytest
import scipy.linalg as sl

from oracle.hqrrp import cpqr_sketch, hqrrp
from oracle.philox import gaussian_block


@pytest.mark.parametrize("rows,s", [(8, 50), (16, 16), (32, 200), (20, 10), (1, 30), (64, 300)])
def test_cpqr_sketch_matches_dgeqp3(rows, s):
    """H3 is the textbook Businger-Golub CPQR: same permutation (swap
    convention included) and the same R as LAPACK dgeqp3 (same dlarfg signs)."""
    Y = np.random.default_rng(rows * 1000 + s).standard_normal((rows, s))
    w = min(rows, s)
    perm, F = cpqr_sketch(Y, w)
    _, Rs, Ps = sl.qr(Y, pivoting=True, mode="economic")
    assert np.array_equal(perm, Ps)
    assert np.max(np.abs(np.triu(F[:w, :]) - Rs[:w, :])) <= 1e-13 * np.linalg.norm(Y)


def test_cpqr_sketch_tie_rule():
    # two equal columns: the lower index wins; then a zero residual (tau = 0)
    Y = np.array([[1.0, 3.0, 3.0], [0.0, 4.0, 4.0]])
    perm, F = cpqr_sketch(Y, 2)
    assert perm[0] == 1
    assert abs(F[0, 0]) == pytest.approx(5.0)


@pytest.mark.parametrize("m,n,b", [(300, 200, 32), (200, 200, 64), (129, 129, 128), (64, 40, 64), (50, 50, 1),
                                   (257, 100, 24)])
def test_hqrrp_invariants(m, n, b):
    A = np.random.default_rng(m + n + b).standard_normal((m, n))
    Q, R, jp = hqrrp(A, b, 11)
    nA = np.linalg.norm(A)
    assert sorted(jp.tolist()) == list(range(n))
    assert np.all(np.tril(R, -1) == 0.0)
    assert np.linalg.norm(A[:, jp] - Q @ R) <= 1e-14 * nA * max(1.0, np.sqrt(n) / 8)
    assert np.linalg.norm(Q.T @ Q - np.eye(m), 2) <= 1e-13
    _, R2, jp2 = hqrrp(A, b, 11, build_q=False)
    assert np.array_equal(jp, jp2) and np.array_equal(R, R2)


def test_hqrrp_orders_orthogonal_columns_by_norm():
    """Columns q_c sigma_c with orthonormal q_c and sigma 1e3 apart: a rank
    revealing QR must pick them in decreasing sigma order, and then
    |diag R| = sigma[jpvt], off-diagonal R = 0 (to rounding)."""
    rng = np.random.default_rng(3)
    m, n, b = 120, 12, 4
    Q0, _ = np.linalg.qr(rng.standard_normal((m, n)))
    sig = 10.0 ** (-3.0 * np.arange(n) / 2)
    order = rng.permutation(n)
    A = Q0 * sig[order]                                  # column c has norm sig[order[c]]
    _, R, jp = hqrrp(A, b, 5)
    assert np.array_equal(order[jp], np.arange(n))      # decreasing sigma
    assert np.allclose(np.abs(np.diag(R)), sig, rtol=1e-12, atol=0)
    off = np.triu(R, 1)
    assert np.max(np.abs(off) / sig[None, :]) <= 1e-12


def test_hqrrp_reveals_exact_rank():
    rng = np.random.default_rng(9)
    m, n, rank, b = 160, 100, 40, 16
    A = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
    _, R, _ = hqrrp(A, b, 2)
    nA = np.linalg.norm(A)
    d = np.abs(np.diag(R))
    assert np.all(d[:rank] > 1e-3 * nA / np.sqrt(n))
    assert np.linalg.norm(R[rank:, rank:]) <= 1e-13 * nA


def test_hqrrp_first_block_pivots_are_dgeqp3_of_the_sketch():
    """H1-H4 composed: the w pivots of step 0 are LAPACK's CPQR pivots of
    Y = G^T A with G the counter-based draw of (seed, 0) (pinned by the Philox
    known-answer tests)."""
    A = np.random.default_rng(4).standard_normal((90, 70))
    b, seed = 16, 123
    _, _, jp = hqrrp(A, b, seed, build_q=False)
    Y = gaussian_block(seed, 0, 90, b).T @ A
    _, _, Ps = sl.qr(Y, pivoting=True, mode="economic")
    assert np.array_equal(jp[:b], Ps[:b])


def test_hqrrp_flops_model():
    # square, b = n: sketch + CPQR + Householder QR of n columns + Q
    from paper_2002_06960_b200.flops import hqrrp_flops
    m = n = b = 64
    fl = hqrrp_flops(m, n, b)
    assert fl == pytest.approx(2 * b * m * n + 2 * b * b * n + 2 * m * n * n - 2 * n ** 3 / 3 + 4 * m * m * n)


def test_hqrrp_partial_is_a_prefix_of_the_full_run():
    """The partial run (K = ceil(k/b) blocks) computes exactly the first K
    steps of the full run; A P = Q R holds with the unreduced trailing block,
    and rho = ||R(k:, k:)||_F is the exact error of the rank-k truncation
    A P ~ Q(:, :k) R(:k, :)."""
    A = np.random.default_rng(21).standard_normal((200, 150))
    Qf, Rf, jf = hqrrp(A, 32, 4)
    for k in (32, 50, 150):
        Q, R, jp, rho = hqrrp(A, 32, 4, k=k)
        K = -(-k // 32) * 32
        assert np.array_equal(jp[:K], jf[:K])
        assert np.array_equal(R[:K, :K], Rf[:K, :K])
        assert np.linalg.norm(A[:, jp] - Q @ R) <= 1e-13 * np.linalg.norm(A)
        assert np.all(R[K:, :K] == 0.0)
        err = np.linalg.norm(A[:, jp] - Q[:, :k] @ R[:k, :])
        assert abs(err - rho) <= 1e-12 * np.linalg.norm(A)
