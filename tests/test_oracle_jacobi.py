"""Pins for oracle O8 (one-sided Jacobi SVD, reading A10)."""
import numpy as np
import pytest

from oracle.jacobi import JacobiNonConvergence, one_sided_jacobi

U = 2.0 ** -53


@pytest.mark.parametrize("b,tri,seed", [(16, False, 0), (64, True, 1), (64, False, 2), (128, True, 3)])
def test_singular_values_match_lapack(b, tri, seed):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((b, b))
    if tri:
        # upper triangular, as on sampled steps, with a graded column scaling
        B = np.triu(B) * np.logspace(0, -3, b)[None, :] + np.diag(np.logspace(0, -3, b))
    Us, d, Vs, sweeps = one_sided_jacobi(B)
    s = np.linalg.svd(B, compute_uv=False)
    assert np.all(np.diff(d) <= 0) and np.all(d >= 0)
    assert np.max(np.abs(d - s)) <= 10 * b * U * s[0]
    assert np.linalg.norm(B - (Us * d) @ Vs.T) <= 1e-13 * np.linalg.norm(B)
    assert np.linalg.norm(Us.T @ Us - np.eye(b), 2) <= 1e-13
    assert np.linalg.norm(Vs.T @ Vs - np.eye(b), 2) <= 1e-13


def test_relative_accuracy_on_graded_matrix():
    # one-sided Jacobi is relatively accurate on column-graded matrices (Demmel-Veselic):
    # B = C D with C well conditioned -> every sigma to a few ulps relative.
    rng = np.random.default_rng(5)
    C = np.linalg.qr(rng.standard_normal((32, 32)))[0] + 0.1 * rng.standard_normal((32, 32))
    D = np.diag(np.logspace(0, -12, 32))
    B = C @ D
    _, d, _, _ = one_sided_jacobi(B)
    # reference: LAPACK on the exactly scaled problem in extended range via QR of C then svd
    s = np.linalg.svd(B, compute_uv=False)
    # LAPACK's bidiagonal SVD is only absolutely accurate; compare the top part tightly and
    # the tail against the product of known factors' bounds
    assert np.max(np.abs(d[:4] - s[:4]) / s[:4]) < 1e-13
    smin_bound = np.linalg.svd(C, compute_uv=False)[-1] * 1e-12
    assert d[-1] >= 0.5 * smin_bound


def test_diag_golden():
    # tests/golden/small_cases.txt: svd_diag
    Us, d, Vs, _ = one_sided_jacobi(np.diag([3.0, 1.0, 2.0]))
    assert np.array_equal(d, [3.0, 2.0, 1.0])
    P = np.eye(3)[:, [0, 2, 1]]
    assert np.array_equal(np.abs(Us), P) and np.array_equal(np.abs(Vs), P)


def test_zero_golden():
    # tests/golden/small_cases.txt: svd_zero
    Us, d, Vs, sweeps = one_sided_jacobi(np.zeros((3, 3)))
    assert np.array_equal(d, [0.0, 0.0, 0.0])
    assert np.array_equal(Us, np.eye(3)) and np.array_equal(Vs, np.eye(3))


def test_rank_deficient_completion_orthogonal():
    rng = np.random.default_rng(9)
    B = np.zeros((6, 6))
    B[:, 1] = rng.standard_normal(6)
    B[:, 4] = rng.standard_normal(6)
    Us, d, Vs, _ = one_sided_jacobi(B)
    assert np.count_nonzero(d) == 2
    assert np.linalg.norm(Us.T @ Us - np.eye(6)) < 1e-14
    assert np.linalg.norm(B - (Us * d) @ Vs.T) < 1e-14 * np.linalg.norm(B)


def test_nonconvergence_reported():
    rng = np.random.default_rng(1)
    with pytest.raises(JacobiNonConvergence):
        one_sided_jacobi(rng.standard_normal((8, 8)), max_sweeps=1)


@pytest.mark.parametrize("b,kind", [(64, "graded"), (128, "gauss_r"), (33, "dense")])
def test_svd_block_transposed_variant(b, kind):
    # svd_block = one-sided Jacobi on B^T (reading A10); same pins as the column variant
    from oracle.jacobi import svd_block
    rng = np.random.default_rng(b)
    B = rng.standard_normal((b, b))
    if kind == "gauss_r":
        B = np.linalg.qr(B)[1]
    elif kind == "graded":
        Q1 = np.linalg.qr(rng.standard_normal((b, b)))[0]
        Q2 = np.linalg.qr(rng.standard_normal((b, b)))[0]
        B = np.linalg.qr((Q1 * 10.0 ** (-8.0 * np.arange(b) / b)) @ Q2.T)[1]
    Us, d, Vs, sweeps = svd_block(B)
    s = np.linalg.svd(B, compute_uv=False)
    assert np.max(np.abs(d - s)) <= 10 * b * U * s[0]
    assert np.linalg.norm(B - (Us * d) @ Vs.T) <= 1e-13 * np.linalg.norm(B)
    assert np.linalg.norm(Us.T @ Us - np.eye(b), 2) <= 1e-13
    assert np.linalg.norm(Vs.T @ Vs - np.eye(b), 2) <= 1e-13
    if kind == "graded":
        assert sweeps <= 12


def test_svd_block_golden_and_zero():
    from oracle.jacobi import svd_block
    Us, d, Vs, _ = svd_block(np.diag([3.0, 1.0, 2.0]))
    assert np.array_equal(d, [3.0, 2.0, 1.0])
    Us, d, Vs, _ = svd_block(np.zeros((3, 3)))
    assert np.array_equal(Us, np.eye(3)) and np.array_equal(Vs, np.eye(3))


def test_svd_block_structurally_rank_deficient_converges():
    # rows of B span a 2-D space: without the negligible-column rule the
    # transposed Jacobi would rotate u-sized null vectors forever
    from oracle.jacobi import svd_block
    rng = np.random.default_rng(9)
    B = np.zeros((6, 6))
    B[:, 1] = rng.standard_normal(6)
    B[:, 4] = rng.standard_normal(6)
    Us, d, Vs, sweeps = svd_block(B)
    assert np.count_nonzero(d) == 2 and sweeps < 10
    assert np.linalg.norm(Us.T @ Us - np.eye(6)) < 1e-14 and np.linalg.norm(Vs.T @ Vs - np.eye(6)) < 1e-14
    assert np.linalg.norm(B - (Us * d) @ Vs.T) < 1e-14 * np.linalg.norm(B)
