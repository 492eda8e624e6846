"""O3/O4 -- unpivoted Householder QR and its compact-WY factor
(TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Paper: step 2 of the randUTV loop, "Compute the unpivoted QR factorization of
T22 V22(:,1:b)" (Sec. 3.1); the construction of V-hat, "Compute the
unpivoted QR factorization of ((T22* T22)^q T22* G)"; FLAME
``[Y, T_V] := unpivoted_QR(Y)`` and ``[[A11;A21], T_U] := unpivoted_QR([A11;A21])``
(P:1330-1331), whose reflectors are kept as "the unit lower
trapezoidal matrices stored below the diagonal" and applied as
X - X W T W* (P:1333-1340).

The paper fixes neither the reflector sign nor the T-factor form (reading A9),
so both follow LAPACK:
* dlarfg: for a column x = (alpha, x'), xi = ||x'||_2.  If xi == 0 then tau = 0
  and H = I (beta = alpha).  Otherwise beta = -sign(alpha) * hypot(alpha, xi)
  with sign(+-0) taken from the IEEE sign bit (copysign), tau = (beta-alpha)/beta,
  v = (1, x'/(alpha-beta)).  H = I - tau v v^T maps x to beta e1.
* dlarft (direct = forward, storev = columnwise): Q = H_1 H_2 ... H_w =
  I - W T W^T with T upper triangular, T[j,j] = tau_j and
  T[0:j, j] = -tau_j T[0:j,0:j] (W[:,0:j]^T w_j).
LAPACK's dlarfg rescaling loop for |beta| < safmin is not reproduced (it only
changes results for inputs below ~1e-292; DESIGN.md lists this).
"""
import math

import numpy as np


def dlarfg(alpha, x):
    """Return (beta, tau, v_tail) for the reflector that annihilates x below alpha."""
    xnorm = math.sqrt(float(np.dot(x, x))) if x.size else 0.0
    if xnorm == 0.0:
        return float(alpha), 0.0, np.zeros_like(x)
    beta = -math.copysign(math.hypot(alpha, xnorm), alpha)
    tau = (beta - alpha) / beta
    v = x / (alpha - beta)
    return beta, tau, v


def householder_qr(P):
    """Unblocked Householder QR of an h x w panel, h >= w (LAPACK dgeqr2 layout).

    Returns (F, tau) with F the factored panel: R on and above the diagonal, the
    reflector tails (unit diagonal implicit) strictly below; tau has w entries.
    Reflector j is applied to the remaining columns one at a time:
    C <- C - tau_j v_j (v_j^T C)  (dlarf).
    """
    F = np.array(P, dtype=np.float64, order="F", copy=True)
    h, w = F.shape
    if h < w:
        raise ValueError("householder_qr expects h >= w")
    tau = np.zeros(w)
    for j in range(w):
        beta, t, v = dlarfg(F[j, j], F[j + 1:, j])
        F[j, j] = beta
        F[j + 1:, j] = v
        tau[j] = t
        if t != 0.0 and j + 1 < w:
            vf = np.concatenate(([1.0], v))
            wrow = vf @ F[j:, j + 1:]
            # F[j:, j+1:] -= t * outer(vf, wrow), the outer product built in the
            # panel's (Fortran) order so the subtraction streams both operands
            O = np.empty((h - j, w - j - 1), order="F")
            np.multiply(vf[:, None], wrow[None, :], out=O)
            O *= t
            F[j:, j + 1:] -= O
    return F, tau


def unit_lower(F):
    """W: the unit lower trapezoidal reflector matrix stored below the diagonal of F."""
    h, w = F.shape
    W = np.tril(F[:, :w], -1)
    W[np.arange(w), np.arange(w)] = 1.0
    return np.asfortranarray(W)


def upper_r(F):
    """R: the w x w upper triangle of the factored panel (exact zeros below)."""
    w = F.shape[1]
    return np.asfortranarray(np.triu(F[:w, :w]))


def larft(W, tau):
    """Forward, columnwise T factor so that H_1...H_w = I - W T W^T (LAPACK dlarft)."""
    w = W.shape[1]
    T = np.zeros((w, w), order="F")
    for j in range(w):
        T[j, j] = tau[j]
        if j > 0 and tau[j] != 0.0:
            T[:j, j] = -tau[j] * (T[:j, :j] @ (W[:, :j].T @ W[:, j]))
    return T
