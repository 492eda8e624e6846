"""Explicit-matrix mini-oracle for tiny inputs (TEST INFRASTRUCTURE ONLY).

Independent of oracle.randutv's compact-WY formulation: every orthogonal factor
is formed as an explicit matrix and the iteration is the paper's Sec. 3.1
equations taken literally:

  V^(i) = diag(I, V22) diag(I, V_SVD, I),  U^(i) = diag(I, U22) diag(I, U_SVD, I)
  T^(i) = U^(i)* T^(i-1) V^(i),  U = U^(0) U^(1) ... ,  V = V^(0) V^(1) ...

V22 is the product H_1 ... H_b of explicit s x s reflectors from the Householder
QR of ((T22* T22)^q T22* G); U22 the product of explicit r x r
reflectors from the QR of T22 V22(:,1:b); the core SVD is LAPACK's
(numpy.linalg.svd) rather than Jacobi, so singular-vector signs may differ from
the oracle's: comparisons against this module use |entries| (a sign flip of
u_j together with v_j of block i multiplies row and column j of T by the same
sign and changes no magnitude).  Final step (s <= b): V22 = I (no sampling, A5).

O(n^4) work per step: keep n <= ~24.
"""
import numpy as np

from .philox import gaussian_block


def _explicit_householder(Mat):
    """QR by explicit reflectors (dlarfg sign convention, reading A9): returns Q = H_1...H_w."""
    X = np.array(Mat, dtype=np.float64, copy=True)
    h, w = X.shape
    Q = np.eye(h)
    for j in range(min(h, w)):
        x = X[j:, j]
        alpha = x[0]
        xnorm = np.sqrt(np.sum(x[1:] ** 2))
        H = np.eye(h)
        if xnorm != 0.0:
            beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            v = np.zeros(h)
            v[j] = 1.0
            v[j + 1:] = x[1:] / (alpha - beta)
            H = np.eye(h) - tau * np.outer(v, v)
        X = H @ X
        Q = Q @ H
    return Q


def randutv_bruteforce(A, b, q, seed):
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    T = A.copy()
    U = np.eye(m)
    V = np.eye(n)
    i = 0
    while i * b < n:
        kk = i * b
        r, s = m - kk, n - kk
        T22 = T[kk:, kk:]
        if s > b:
            G = gaussian_block(seed, i, r, b)
            Y = T22.T @ G
            for _ in range(q):
                Y = T22.T @ (T22 @ Y)
            V22 = _explicit_householder(Y)
            w = b
        else:
            V22 = np.eye(s)
            w = s
        U22 = _explicit_householder((T22 @ V22)[:, :w])
        core = (U22[:, :w].T @ T22 @ V22[:, :w])
        Usvd, d, VsvdT = np.linalg.svd(core)
        Vi = np.eye(n)
        Vi[kk:, kk:] = V22
        Vs = np.eye(n)
        Vs[kk:kk + w, kk:kk + w] = VsvdT.T
        Vi = Vi @ Vs
        Ui = np.eye(m)
        Ui[kk:, kk:] = U22
        Us = np.eye(m)
        Us[kk:kk + w, kk:kk + w] = Usvd
        Ui = Ui @ Us
        T = Ui.T @ T @ Vi
        U = U @ Ui
        V = V @ Vi
        i += 1
    return {"U": U, "T": T, "V": V}
