"""O8 -- SVD of the small core block by one-sided (Hestenes) Jacobi
(TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Paper: step 3 of the randUTV loop, "Compute the SVD of (U22(:,1:b))* T22
V22(:,1:b) = U_SVD D V_SVD*" (Sec. 3.1); FLAME
``[A11, U_SVD, V_SVD] := SVD(A11)`` (Fig. fig:FLArandutv); task
``Svd_of_block`` (Fig. fig:analyzer).  The paper does not name the
SVD algorithm (reading A10); this oracle uses the textbook one-sided Jacobi
method with the cyclic-by-rows pair order:

    X := B, V := I.  For each pair (p < q) in row-cyclic order:
      alpha = x_p.x_p, beta = x_q.x_q, gamma = x_p.x_q
      if |gamma| > tol*sqrt(alpha*beta):
        zeta = (beta - alpha) / (2 gamma)
        t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),  c = 1/sqrt(1+t^2), s = c t
        (x_p, x_q) <- (c x_p - s x_q, s x_p + c x_q), same for (v_p, v_q)
    Stop after the first sweep with no rotation; more than ``max_sweeps``
    sweeps is non-convergence.
    d_j = ||x_j||, U(:,j) = x_j / d_j; columns with d_j == 0 are completed by
    Gram-Schmidt of e_1, e_2, ... against the columns already present.
    Sort d descending (stable), permuting U and V alike.

tol = sqrt(b) * 2^-53 (LAPACK dgesvj's sqrt(m)*eps), max_sweeps = 30.
Columns with ||x|| <= nu = b 2^-53 ||B||_F are numerically null: pairs that
involve one are not rotated and their d is set to 0 (then completed).  Without
this rule a rank-deficient block never converges: rounding leaves more
u-sized "null" vectors than the null space has dimensions, and no rotation can
make them mutually orthogonal under the relative test.
The rotation annihilates the (p,q) Gram entry exactly in exact arithmetic:
gamma' = cs(alpha - beta) + (c^2 - s^2) gamma = 0.

``svd_block`` (what randUTV calls, reading A10) runs the method on B^T, i.e. it
orthogonalises the ROWS of B: B^T W = Q diag(d) gives B = W diag(d) Q^T, so
U_SVD = W (the accumulated rotations) and V_SVD = Q.  On the rank-revealing,
row-graded R of a randUTV step this converges in far fewer sweeps than
orthogonalising the columns (e.g. 8-9 vs 21-25 sweeps on a 64/128 block whose
singular values span 8 decades) -- the transposition trick of Drmac & Veselic.
"""
import math

import numpy as np


class JacobiNonConvergence(RuntimeError):
    pass


def jacobi_tol(b):
    return math.sqrt(b) * 2.0 ** -53


def negligible_norm(B):
    """nu = n 2^-53 ||B||_F: columns this short are numerical zeros (not rotated, d := 0)."""
    return B.shape[1] * 2.0 ** -53 * math.sqrt(float(np.sum(np.asarray(B) ** 2)))


def one_sided_jacobi(B, tol=None, max_sweeps=30):
    """Return (Us, d, Vs, sweeps) with B = Us diag(d) Vs^T, d >= 0 descending."""
    X = np.array(B, dtype=np.float64, order="F", copy=True)
    nr, n = X.shape
    V = np.eye(n, order="F")
    if tol is None:
        tol = jacobi_tol(n)
    nu2 = negligible_norm(X) ** 2
    sweeps = 0
    converged = n <= 1
    while not converged:
        if sweeps >= max_sweeps:
            raise JacobiNonConvergence(f"one-sided Jacobi: no convergence in {max_sweeps} sweeps")
        sweeps += 1
        rotated = False
        for p in range(n - 1):
            for q in range(p + 1, n):
                xp = X[:, p]
                xq = X[:, q]
                alpha = float(xp @ xp)
                beta = float(xq @ xq)
                gamma = float(xp @ xq)
                if alpha > nu2 and beta > nu2 and abs(gamma) > tol * math.sqrt(alpha * beta):
                    rotated = True
                    zeta = (beta - alpha) / (2.0 * gamma)
                    t = math.copysign(1.0, zeta) / (abs(zeta) + math.hypot(1.0, zeta))
                    c = 1.0 / math.sqrt(1.0 + t * t)
                    s = c * t
                    xp0 = xp.copy()
                    X[:, p] = c * xp0 - s * xq
                    X[:, q] = s * xp0 + c * xq
                    vp0 = V[:, p].copy()
                    vq0 = V[:, q].copy()
                    V[:, p] = c * vp0 - s * vq0
                    V[:, q] = s * vp0 + c * vq0
        converged = not rotated
    d = np.sqrt(np.einsum("ij,ij->j", X, X))
    d[d * d <= nu2] = 0.0          # numerically null columns -> exact zeros (completed below)
    U = np.zeros((nr, n), order="F")
    for j in range(n):
        if d[j] != 0.0:
            U[:, j] = X[:, j] / d[j]
    _complete_basis(U, d)
    order = sorted(range(n), key=lambda j: -d[j])  # Python's sort is stable
    return (np.asfortranarray(U[:, order]), d[order].copy(),
            np.asfortranarray(V[:, order]), sweeps)


def svd_block(B, tol=None, max_sweeps=30):
    """SVD of the small core block (O8): one-sided Jacobi on B^T; returns (Us, d, Vs, sweeps)."""
    Q, d, W, sweeps = one_sided_jacobi(np.asarray(B).T, tol=tol, max_sweeps=max_sweeps)
    return W, d, Q, sweeps


def _complete_basis(U, d):
    """Fill the columns with d_j == 0 by Gram-Schmidt of e_1, e_2, ... (twice)."""
    nr, n = U.shape
    e = 0
    for j in range(n):
        if d[j] != 0.0:
            continue
        while True:
            if e >= nr:
                raise RuntimeError("cannot complete basis")
            x = np.zeros(nr)
            x[e] = 1.0
            e += 1
            have = [i for i in range(n) if d[i] != 0.0 or np.any(U[:, i])]
            for _ in range(2):
                for i in have:
                    x -= (U[:, i] @ x) * U[:, i]
            nx = math.sqrt(float(x @ x))
            if nx > 0.5:
                U[:, j] = x / nx
                break
