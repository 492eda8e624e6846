"""Pins for oracle O3/O4 (Householder QR + compact-WY T factor, reading A9).

Library pin: scipy.linalg.qr(mode='raw') returns LAPACK dgeqrf's factored panel
and tau; the oracle's unblocked column loop must reproduce them (same dlarfg
convention).  scipy's explicit Q (dorgqr) pins the T factor.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle.householder import dlarfg, householder_qr, larft, unit_lower, upper_r

U = 2.0 ** -53


@pytest.mark.parametrize("h,w,seed", [(5, 5, 0), (40, 7, 1), (300, 64, 2), (129, 33, 3), (8, 1, 4)])
def test_qr_matches_lapack_dgeqrf(h, w, seed):
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((h, w))
    P[0, 0] = -abs(P[0, 0])  # exercise both signs of alpha
    F, tau = householder_qr(P)
    (Fl, taul), _ = sla.qr(P, mode="raw")
    kappa = np.linalg.cond(P)
    tol = 50 * kappa * h * U
    assert np.max(np.abs(tau - taul)) <= tol
    assert np.max(np.abs(np.triu(F[:w]) - np.triu(Fl[:w]))) <= tol * np.linalg.norm(P)
    assert np.max(np.abs(np.tril(F, -1) - np.tril(Fl, -1))) <= tol


@pytest.mark.parametrize("h,w", [(50, 10), (200, 64), (64, 64)])
def test_wy_equals_explicit_reflector_product_and_lapack_q(h, w):
    rng = np.random.default_rng(h + w)
    P = rng.standard_normal((h, w))
    F, tau = householder_qr(P)
    W = unit_lower(F)
    T = larft(W, tau)
    Q = np.eye(h) - W @ T @ W.T
    # brute force: multiply the explicit reflectors H_1 ... H_w
    Qb = np.eye(h)
    for j in range(w):
        v = W[:, j]
        Qb = Qb @ (np.eye(h) - tau[j] * np.outer(v, v))
    assert np.max(np.abs(Q - Qb)) <= 1e-15 * 10 * w
    # LAPACK's explicit Q (dorgqr from dgeqrf)
    Ql, Rl = sla.qr(P, mode="full")
    assert np.max(np.abs(Q - Ql)) <= 1e-13
    # QR reproduces the panel, Q orthogonal, T upper triangular
    R = upper_r(F)
    assert np.linalg.norm(P - Q[:, :w] @ R) <= 10 * h * U * np.linalg.norm(P)
    assert np.linalg.norm(Q.T @ Q - np.eye(h), 2) <= 10 * h * U
    assert np.all(np.tril(T, -1) == 0)


def test_qr_3_4_golden():
    # tests/golden/small_cases.txt: qr_3_4
    beta, tau, v = dlarfg(3.0, np.array([4.0]))
    assert beta == -5.0 and tau == pytest.approx(1.6, rel=1e-15) and v[0] == pytest.approx(0.5, rel=1e-15)
    F, t = householder_qr(np.array([[3.0], [4.0]]))
    assert abs(F[0, 0]) == 5.0


def test_identity_and_zero_columns_give_tau_zero():
    F, tau = householder_qr(np.eye(6)[:, :4])
    assert np.all(tau == 0.0)
    assert np.array_equal(upper_r(F), np.eye(4))
    Z = np.zeros((5, 3))
    Z[:, 1] = 1.0
    F, tau = householder_qr(Z)
    assert tau[0] == 0.0 and tau[2] == 0.0 and tau[1] != 0.0
    W = unit_lower(F)
    T = larft(W, tau)
    assert T[0, 0] == 0.0 and np.all(T[:, 0] == 0.0)


def test_negative_zero_alpha_sign_follows_copysign():
    b1, _, _ = dlarfg(0.0, np.array([1.0]))
    b2, _, _ = dlarfg(-0.0, np.array([1.0]))
    assert b1 == -1.0 and b2 == 1.0
