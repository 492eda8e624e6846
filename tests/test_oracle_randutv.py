"""Pins for the full oracle randUTV (O1-O11), against things other than itself:
the explicit-matrix mini-oracle (paper Sec. 3.1 equations taken literally),
LAPACK's SVD in the cases where randUTV reduces to it, closed forms of the c1
spectrum, exact invariants (orthogonality, triangularity, norms), and the
identity rho = ||A - A_k||_F of the truncated variant.
"""
import math

import numpy as np
import pytest

from oracle.bruteforce import randutv_bruteforce
from oracle.randutv import orthogonality_error, randutv, reconstruction_error
from paper_2002_06960_b200.inputs import make_numpy, sigma_powspec

U = 2.0 ** -53


@pytest.fixture(scope="module")
def c1():
    A = make_numpy("powspec", 512, 512, cfg_index=1)
    out = randutv(A, 64, 2, 2001)
    return A, out


@pytest.mark.parametrize("m,n,b,q", [(12, 12, 4, 1), (14, 10, 3, 2), (9, 9, 2, 0), (10, 7, 7, 1),
                                     (8, 8, 8, 0), (11, 11, 1, 1), (16, 13, 5, 2), (13, 13, 20, 1)])
def test_matches_explicit_matrix_bruteforce(m, n, b, q):
    rng = np.random.default_rng(m * 100 + n * 10 + b)
    A = rng.standard_normal((m, n))
    o = randutv(A, b, q, 77)
    bf = randutv_bruteforce(A, b, q, 77)
    # singular-vector signs may differ (LAPACK vs Jacobi); magnitudes are invariant
    for key in ("T", "U", "V"):
        assert np.max(np.abs(np.abs(o[key]) - np.abs(bf[key]))) <= 1e-13, key


def test_c1_exact_invariants(c1):
    A, o = c1
    Uo, T, V = o["U"], o["T"], o["V"]
    assert reconstruction_error(A, Uo, T, V) <= 1e-13
    assert orthogonality_error(Uo) <= 1e-13
    assert orthogonality_error(V) <= 1e-13
    assert np.all(np.tril(T, -1) == 0.0)                 # exactly triangular (A15)
    assert abs(np.linalg.norm(T) / np.linalg.norm(A) - 1) <= 1e-14
    assert np.all(np.diag(T) >= 0)                       # A14


def test_c1_log_det_closed_form(c1):
    # tests/golden/small_cases.txt: c1_logdet = -2048
    _, o = c1
    s = np.sum(np.log10(np.abs(np.diag(o["T"]))))
    assert abs(s - (-2048.0)) <= 1e-6


def test_c1_weyl_log_majorisation(c1):
    # diag(T) are T's eigenvalues; |lambda| are log-majorised by the singular values
    _, o = c1
    t = np.sort(np.abs(np.diag(o["T"])))[::-1]
    sig = sigma_powspec(512)
    assert np.all(np.cumsum(np.log(t)) <= np.cumsum(np.log(sig)) + 1e-9)


def test_c1_diag_tracks_singular_values(c1):
    # calibrated (not from the paper): P:227-236 says q = 1, 2 get "within striking
    # distance" of the SVD and diag(T) approximates the singular values.
    _, o = c1
    rel = np.abs(np.abs(np.diag(o["T"])) / sigma_powspec(512) - 1)
    assert np.median(rel) <= 1e-2 and np.max(rel) <= 0.3


@pytest.mark.parametrize("k", [64, 128])
def test_c1_rank_k_error_near_optimal_and_truncated_agrees(c1, k):
    A, o = c1
    sig = sigma_powspec(512)
    Ak = o["U"][:, :k] @ o["T"][:k, :] @ o["V"].T
    e2 = np.linalg.norm(A - Ak, 2)
    ratio = e2 / sig[k]
    assert 1.0 - 1e-9 <= ratio <= 1.5                    # Eckart-Young and the calibrated bound
    rho_full = np.linalg.norm(o["T"][k:, k:])
    assert abs(np.linalg.norm(A - Ak) - rho_full) <= 1e-12 * np.linalg.norm(A)
    tr = randutv(A, 64, 2, 2001, k=k)
    Ak_t = tr["Uk"] @ tr["Tk"] @ tr["V"].T
    assert np.linalg.norm(Ak_t - Ak) <= 1e-12 * np.linalg.norm(A)
    assert abs(tr["rho"] - rho_full) <= 1e-12 * np.linalg.norm(A)
    assert abs(tr["rho"] - np.linalg.norm(A - Ak_t)) <= 1e-12 * np.linalg.norm(A)


def test_b_at_least_n_reduces_to_svd():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((40, 30))
    o = randutv(A, 30, 1, 5)
    s = np.linalg.svd(A, compute_uv=False)
    assert np.max(np.abs(np.abs(np.diag(o["T"])) - s)) <= 1e-13 * s[0]
    assert reconstruction_error(A, o["U"], o["T"], o["V"]) <= 1e-13


def test_exact_low_rank_within_first_block():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((96, 5))
    Y = rng.standard_normal((96, 5))
    A = X @ Y.T
    o = randutv(A, 16, 1, 9)
    s = np.linalg.svd(A, compute_uv=False)
    d = np.abs(np.diag(o["T"]))
    assert np.max(np.abs(d[:5] - s[:5]) / s[:5]) <= 1e-12
    assert np.max(d[5:]) <= 1e-13 * s[0]
    assert np.linalg.norm(o["T"][16:, 16:]) <= 1e-13 * s[0]


def test_tall_and_ragged_and_thin_u():
    rng = np.random.default_rng(6)
    A = rng.standard_normal((150, 70))
    o = randutv(A, 16, 1, 11)
    assert reconstruction_error(A, o["U"], o["T"], o["V"]) <= 1e-13
    assert np.all(np.tril(o["T"], -1) == 0.0)
    assert np.all(o["T"][70:, :] == 0.0)
    th = randutv(A, 16, 1, 11, thin_u=True)
    assert np.max(np.abs(th["U"] - o["U"][:, :70])) <= 1e-13
    assert np.array_equal(th["T"], o["T"])
    tr = randutv(A, 16, 1, 11, k=40, thin_u=True)
    Ak = tr["Uk"] @ tr["Tk"] @ tr["V"].T
    assert abs(np.linalg.norm(A - Ak) - tr["rho"]) <= 1e-12 * np.linalg.norm(A)
    assert orthogonality_error(tr["Uk"]) <= 1e-13


def test_q_improves_rank_revealing():
    A = make_numpy("powspec", 256, 256, cfg_index=1)
    sig = sigma_powspec(256)
    errs = {}
    for q in (0, 2):
        o = randutv(A, 32, q, 3)
        errs[q] = np.mean(np.abs(np.abs(np.diag(o["T"])) / sig - 1))
    assert errs[2] < errs[0]


def test_zero_matrix_and_b1():
    Z = np.zeros((10, 6))
    o = randutv(Z, 4, 1, 1)
    assert np.all(o["T"] == 0.0)
    assert orthogonality_error(o["U"]) <= 1e-15 and orthogonality_error(o["V"]) <= 1e-15
    rng = np.random.default_rng(8)
    A = rng.standard_normal((9, 9))
    o = randutv(A, 1, 1, 2)
    assert reconstruction_error(A, o["U"], o["T"], o["V"]) <= 1e-13
    assert abs(np.prod(np.abs(np.diag(o["T"]))) / abs(np.linalg.det(A)) - 1) <= 1e-12


def test_seed_determinism():
    rng = np.random.default_rng(10)
    A = rng.standard_normal((40, 40))
    o1 = randutv(A, 8, 1, 123)
    o2 = randutv(A, 8, 1, 123)
    o3 = randutv(A, 8, 1, 124)
    assert np.array_equal(o1["T"], o2["T"])
    assert not np.array_equal(o1["T"], o3["T"])


def test_invalid_arguments():
    with pytest.raises(ValueError):
        randutv(np.zeros((3, 5)), 2, 1, 0)
    with pytest.raises(ValueError):
        randutv(np.zeros((5, 5)), 0, 1, 0)


# ---------------------------------------------------------------- NEXT-4: re-orthonormalised power steps
def test_orth_matches_lapack_q():
    """_orth is the explicit Householder Q: identical (signs included, same
    dlarfg convention) to LAPACK dgeqrf + dorgqr via numpy."""
    from oracle.randutv import _orth
    X = np.random.default_rng(8).standard_normal((200, 24))
    Q = _orth(X)
    Qn, _ = np.linalg.qr(X)
    assert np.max(np.abs(Q - Qn)) <= 1e-14
    assert np.allclose(np.tril(Q.T @ X, -1), 0.0, atol=1e-13)


def test_reorth_same_span_on_well_conditioned():
    # exact arithmetic: the same span, hence the same T up to rounding
    A = np.asfortranarray(np.random.default_rng(5).standard_normal((300, 200)))
    o1 = randutv(A, 32, 2, 5)
    o2 = randutv(A, 32, 2, 5, reorth=True)
    d1, d2 = np.abs(np.diag(o1["T"])), np.abs(np.diag(o2["T"]))
    assert np.max(np.abs(d1 - d2) / d1) <= 1e-12
    assert np.linalg.norm(A - o2["U"] @ o2["T"] @ o2["V"].T) <= 1e-13 * np.linalg.norm(A)


def test_reorth_resolves_graded_spectrum():
    """sigma_j = 10^(-j/8), q = 3: the literal products (A8) push directions
    below eps^(1/7) of a block's top singular value under rounding, and
    |T_jj| / sigma_j strays by more than 10x; re-orthonormalised power steps
    keep it within [0.5, 2] down to sigma = 1e-16."""
    rng = np.random.default_rng(0)
    n = 256
    U0, _ = np.linalg.qr(rng.standard_normal((n, n)))
    V0, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = 10.0 ** (-np.arange(n) / 8)
    A = np.asfortranarray((U0 * sig) @ V0.T)
    lit = np.abs(np.diag(randutv(A, 32, 3, 5, build_uv=False)["T"]))[:n // 2] / sig[:n // 2]
    ro = np.abs(np.diag(randutv(A, 32, 3, 5, build_uv=False, reorth=True)["T"]))[:n // 2] / sig[:n // 2]
    assert ro.min() >= 0.5 and ro.max() <= 2.0
    assert lit.min() < 0.1 or lit.max() > 10.0


# ---------------------------------------------------------------- NEXT-4: oversampling (reading A28)
def test_oversample_zero_is_the_literal_scheme():
    A = np.random.default_rng(3).standard_normal((90, 70))
    o0, o1 = randutv(A, 16, 1, 9), randutv(A, 16, 1, 9, oversample=0)
    for key in ("T", "U", "V"):
        assert np.array_equal(o0[key], o1[key])


@pytest.mark.parametrize("m,n,b", [(64, 64, 16), (80, 48, 12), (50, 50, 7)])
def test_oversample_spanning_sample_reduces_to_svd(m, n, b):
    """Closed form: when b + p >= s at every step the sample spans the whole
    trailing row space, the Rayleigh-Ritz selection picks exactly its top-b right
    singular subspace, and |diag T| = the singular values of A in order (LAPACK)."""
    A = np.random.default_rng(m + n + b).standard_normal((m, n))
    o = randutv(A, b, 0, 11, oversample=n)
    s = np.linalg.svd(A, compute_uv=False)
    assert np.max(np.abs(np.abs(np.diag(o["T"])) - s)) <= 1e-13 * s[0]
    assert reconstruction_error(A, o["U"], o["T"], o["V"]) <= 1e-13
    assert orthogonality_error(o["U"]) <= 1e-13 and orthogonality_error(o["V"]) <= 1e-13


def test_oversample_select_is_rayleigh_ritz():
    """_select returns an orthonormal basis of the b-dimensional subspace of
    span(Y) on which A_t is largest: ||A_t Y_hat||_F^2 equals the sum of the top
    b squared singular values of A_t Q_Y (numpy SVD)."""
    from oracle.randutv import _orth, _select
    rng = np.random.default_rng(5)
    At = rng.standard_normal((120, 90)) * (0.9 ** np.arange(90))
    Y = At.T @ rng.standard_normal((120, 24))
    Yh = _select(At, Y, 16)
    assert orthogonality_error(Yh) <= 1e-14
    sv = np.linalg.svd(At @ _orth(Y), compute_uv=False)
    assert abs(np.linalg.norm(At @ Yh) ** 2 - np.sum(sv[:16] ** 2)) <= 1e-12 * np.sum(sv[:16] ** 2)
    # Y_hat lies in span(Y)
    Q = _orth(Y)
    assert np.linalg.norm(Yh - Q @ (Q.T @ Yh)) <= 1e-13


def test_oversample_improves_range_finder_on_c1():
    """q = 0 on c1: the rank-64 residual decreases with p and reaches the
    Eckart-Young optimum sqrt(sum_{j > 64} sigma_j^2) within 1 % at p = b."""
    A = make_numpy("powspec", 512, 512, cfg_index=1)
    sig = sigma_powspec(512)
    opt = math.sqrt(float(np.sum(sig[64:] ** 2)))
    rhos = [randutv(A, 64, 0, 2001, k=64, thin_u=True, oversample=p)["rho"] for p in (0, 8, 32, 64)]
    assert all(a >= b for a, b in zip(rhos, rhos[1:]))
    assert rhos[0] > 1.2 * opt and rhos[-1] <= 1.01 * opt


def test_oversample_invariants_ragged_tall():
    A = np.random.default_rng(8).standard_normal((150, 101))
    o = randutv(A, 24, 1, 4, oversample=10)
    assert reconstruction_error(A, o["U"], o["T"], o["V"]) <= 1e-13
    assert orthogonality_error(o["U"]) <= 1e-13 and orthogonality_error(o["V"]) <= 1e-13
    assert np.all(np.tril(o["T"], -1) == 0.0)
    ot = randutv(A, 24, 1, 4, oversample=10, k=48, thin_u=True)
    assert abs(ot["rho"] - np.linalg.norm(o["T"][48:, 48:])) <= 1e-12 * np.linalg.norm(A)
