"""HQRRP -- the blocked randomized column-pivoted Householder QR
(TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Follows Sec. 2 of the paper ("Partial rank-revealing QR factorization",
P:252-362) step by step.  A (m x n, m >= n) is factored as A = Q R P^*
 in ceil(n/b) blocked steps; R^(0) = A, Q^(0) = I, P^(0) = I
(P:285-290).  Step i (k = i b, r = m - k trailing rows, s = n - k trailing
columns, w = min(b, s)):

  H1  G^(i): b x (m - ib) standard normal.  Reading A26: G^(i) is
      the transpose of randUTV's draw for (seed, i) (oracle.philox, same
      counters), so both methods share one generator.
  H2  Y^(i) = G^(i) R22^(i-1)   (b x s)
  H3  w steps of the traditional CPQR of Y^(i): Y P22 = W_trash S_trash
      (P:337-339).  Reading A27: "traditional" = Businger-Golub with
      Householder reflectors (dlarfg convention, oracle.householder): at step j
      the pivot is the remaining column with the largest norm of rows j:b
      (norms recomputed, not downdated; exact ties -> the lowest column
      index of Y), swapped into position j (LAPACK dgeqp3's swap
      convention for the permutation of the other columns).
  H4  P^(i) = diag(I, P22): the columns k:n of R (all m rows) are
      permuted; jpvt records the original column index of every position.
  H5  unpivoted QR of the first w permuted columns (rows k:m):
      R22 P22(:, 1:w) = Q22 R22(:, 1:w), R11 := R (strict lower
      part 0), the rows below := 0; the reflectors W, T (compact WY,
      oracle.householder.larft) give Q^(i) = diag(I, Q22).
  H6  R(k:m, k+w:n) := Q22^* R(k:m, k+w:n);  Q(:, k:m) := Q(:, k:m) Q22
      (R^(i) = Q^(i)* R^(i-1) P^(i), Q = Q^(0) Q^(1) ...).

The paper's downdated-sketch variant (Remark) is not used by its
primary implementation and not here either.
"""
import numpy as np

from .householder import dlarfg, householder_qr, larft, unit_lower, upper_r
from .philox import gaussian_block


def cpqr_sketch(Y, steps):
    """H3: `steps` steps of Businger-Golub CPQR of Y (rows x s).

    Returns (perm, F): perm[j] = the column of Y in position j after the swaps;
    F = the partially factored, permuted Y (R above the diagonal of the first
    `steps` columns, reflector tails below, the updated rest to the right).
    """
    F = np.array(Y, dtype=np.float64, order="F", copy=True)
    rows, s = F.shape
    perm = np.arange(s)
    for j in range(steps):
        # squared norms of rows j: of the remaining columns (positions j:s)
        nrm2 = np.sum(F[j:, j:] ** 2, axis=0)
        best = np.max(nrm2)
        cand = np.nonzero(nrm2 == best)[0] + j
        p = cand[np.argmin(perm[cand])]          # exact tie: lowest original index
        if p != j:
            F[:, [j, p]] = F[:, [p, j]]
            perm[[j, p]] = perm[[p, j]]
        beta, tau, v = dlarfg(F[j, j], F[j + 1:, j])
        F[j, j] = beta
        F[j + 1:, j] = v
        if tau != 0.0 and j + 1 < s:
            vf = np.concatenate(([1.0], v))
            wrow = vf @ F[j:, j + 1:]
            F[j:, j + 1:] -= tau * np.outer(vf, wrow)
    return perm, F


def hqrrp(A, b, seed, build_q=True, record=None, k=None):
    """Oracle HQRRP of A (m x n, m >= n): returns (Q, R, jpvt) with
    A[:, jpvt] = Q R, Q (m x m) orthogonal (None if not build_q), R upper
    trapezoidal, jpvt a permutation of 0..n-1.  `record`, if a list, receives
    per step the dict {k, w, perm} (perm: positions k:n after H4, as indices
    into the columns k:n before it).

    k (partial factorisation, the section's "partial rank-revealing QR",
    P:252-262): stop after K = ceil(k / b) blocks; then A[:, jpvt] = Q R still
    holds with R(K b:m, K b:n) the unreduced trailing block, and the rank-k
    truncation error is rho = ||R(k:m, k:n)||_F, returned as a 4th value."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    if m < n:
        raise ValueError("hqrrp expects m >= n")
    if b < 1:
        raise ValueError("b >= 1")
    b = min(b, n)                                         # 1 <= b <= n
    R = np.array(A, order="F", copy=True)
    Q = np.eye(m, order="F") if build_q else None
    jpvt = np.arange(n)
    i = 0
    kstop = n if k is None else min(n, -(-int(k) // b) * b)
    if k is not None and not (1 <= k <= n):
        raise ValueError("need 1 <= k <= n")
    ktrunc = k
    for k in range(0, kstop, b):
        r, s = m - k, n - k
        w = min(b, s)
        # H1, H2
        G = gaussian_block(seed, i, r, b)                 # (m - ib) x b; G^(i) = G^T
        Y = G.T @ R[k:, k:]                               # b x s
        # H3, H4
        perm, _ = cpqr_sketch(Y, w)
        R[:, k:] = R[:, k:][:, perm]
        jpvt[k:] = jpvt[k:][perm]
        if record is not None:
            record.append({"k": k, "w": w, "perm": perm.copy()})
        # H5
        F, tau = householder_qr(R[k:, k:k + w])
        W = unit_lower(F)
        Tq = larft(W, tau)
        R[k:k + w, k:k + w] = upper_r(F)
        R[k + w:, k:k + w] = 0.0
        # H6
        if k + w < n:
            R[k:, k + w:] -= W @ (Tq.T @ (W.T @ R[k:, k + w:]))
        if build_q:
            Q[:, k:] -= ((Q[:, k:] @ W) @ Tq) @ W.T
        i += 1
    if ktrunc is not None:
        return Q, R, jpvt, float(np.linalg.norm(R[ktrunc:, ktrunc:]))
    return Q, R, jpvt

