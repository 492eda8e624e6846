"""randUTV -- the blocked randomized UTV factorization with power iteration
(TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Follows Sec. 3.1 of the paper step by step, in the order of the FLAME loop
(Fig. fig:FLArandutv) and of the task list of Fig. fig:analyzer
(P:1529-1594), with the readings of DESIGN.md:

  init      T := A, U := I_m, V := I_n
  loop      i = 0, 1, ... while columns remain, k = i b,       (A1: n-guard)
            r = m - k trailing rows, s = n - k trailing columns
  sampled step (s > b):
   O1  G := N(0,1)^{r x b} (oracle.philox)
   O2  Y := A_t^T G; q times { Z := A_t Y; Y := A_t^T Z },     (
       A_t = T[k:m, k:n], the literal product (A8)               A8: no re-orthonormalisation)
   O3/O4 [W_V, tau_V, T_V] := QR(Y)
   O5  T[0:m, k:n] -= (T[0:m,k:n] W_V) T_V W_V^T  (all m rows, A2)
       V[0:n, k:n] -= (V[0:n,k:n] W_V) T_V W_V^T
   O6  [W_U, tau_U, T_U] := QR(T[k:m, k:k+b]); T[k:k+b,k:k+b] := R (strict lower 0),
       T[k+b:m, k:k+b] := 0                                     (Keep_upper_triang,
                                                                 Set_to_zero P:1577-1582)
   O7  T[k:m, k+b:n] -= W_U T_U^T (W_U^T T[k:m, k+b:n])  (A3)
       U[0:m, k:m]   -= (U[0:m,k:m] W_U) T_U W_U^T
   O8  R = U_s diag(d) V_s^T (oracle.jacobi.svd_block)
   O9  T[k:k+b,k:k+b] := diag(d); T[0:k, k:k+b] := T[0:k,k:k+b] V_s;
       T[k:k+b, k+b:n] := U_s^T T[k:k+b, k+b:n]; U[:,k:k+b] := U[:,k:k+b] U_s;
       V[:,k:k+b] := V[:,k:k+b] V_s
  final step (s <= b; A5: no sampling, Fig. fig:analyzer's last tasks P:1589-1594)
   O10 if r > s: O6 with width s and the U update of O7, then O8 on R;
       else O8 on the dense s x s block T[k:n, k:n];  then O9 with b := s.
  O11 outputs: full -> (U, T, V); truncated (K = ceil(k/b) sampled steps, no O10)
       -> (U[:, :k], T[:k, :], V, rho = ||T[k:m, k:n]||_F = ||A - A_k||_F)

Thin U (A12): instead of the m x m forward accumulation, the left transforms
(k_j, W_U, T_U, U_s) are recorded and U(:, :c) = U^(1) ... U^(p) [I_c; 0] is
formed backward: X := [I_c; 0]; for j = p..1: X[k_j:k_j+b_j, :] := U_s X[...];
X[k_j:m, :] -= W_U T_U (W_U^T X[k_j:m, :]).
"""
import math

import numpy as np

from .householder import householder_qr, larft, unit_lower, upper_r
from .jacobi import svd_block
from .philox import gaussian_block


def _mm(A, B):
    """A @ B written in Fortran order (np.matmul into an F-ordered out): the
    rank-b products below are subtracted from Fortran-ordered views, and a
    C-ordered temporary would make that subtraction walk memory transposed
    (50x slower at the full sizes).  Same products, same BLAS call."""
    out = np.empty((A.shape[0], B.shape[1]), order="F")
    return np.matmul(A, B, out=out)


def sampled_steps(n, b):
    """Number of sampled steps (those with s = n - i b > b)."""
    return max(0, -(-(n - b) // b)) if n > b else 0


def randutv(A, b, q, seed, build_uv=True, k=None, thin_u=False, record=None, reorth=False, overwrite_a=False,
            oversample=0):
    """Oracle randUTV of A (m x n, m >= n).

    Parameters
    ----------
    b, q, seed : block size, power steps, 64-bit seed of G (O1)
    build_uv   : accumulate U and V
    k          : if given, the truncated variant: K = ceil(k/b) sampled steps, no
                 final step (if K reaches the final step the full factorisation is
                 run and truncated)
    thin_u     : form U by backward accumulation (economy m x n, or m x k truncated)
    record     : optional dict; receives per-step diagnostics (Y, tau, d, ...)
    reorth     : re-orthonormalise the sample between power steps (SURVEY §8(f)
                 NEXT-4, the alternative to reading A8; see _sample)
    oversample : p >= 0 extra sample columns with Rayleigh-Ritz selection of the
                 b directions (reading A28; see _select)
    overwrite_a: T is A itself (A must be a Fortran-ordered float64 array) -- the
                 paper's in-place factorisation ("T := A"); saves one
                 copy of A for the full-size parity tests (17-34 GB)

    Returns dict with keys U, T, V (full) or Uk, Tk, V, rho (truncated).
    """
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    if m < n:
        raise ValueError("randUTV assumes m >= n (P:532)")
    if b < 1 or q < 0 or oversample < 0:
        raise ValueError("need b >= 1, q >= 0, oversample >= 0")
    if overwrite_a:
        if not (A.flags.f_contiguous and A.dtype == np.float64):
            raise ValueError("overwrite_a needs a Fortran-ordered float64 A")
        T = A
    else:
        T = np.array(A, order="F", copy=True)
    forward_u = build_uv and not thin_u
    U = np.eye(m, order="F") if forward_u else None
    V = np.eye(n, order="F") if build_uv else None
    lefts = []  # (k, W_U, T_U, U_s) for thin U
    nsamp = sampled_steps(n, b)
    K = nsamp
    truncated = k is not None
    if truncated:
        if not (1 <= k <= n):
            raise ValueError("need 1 <= k <= n")
        K = -(-k // b)
        if K > nsamp:
            truncated_full = True
            K = nsamp
        else:
            truncated_full = False
    i = 0
    while True:
        kk = i * b
        r, s = m - kk, n - kk
        if s <= 0:
            break
        if s > b:
            if i >= K:
                break
            _sampled_step(T, U, V, lefts, kk, b, q, seed, i, thin_u and build_uv, record, reorth, oversample)
        else:
            if truncated and not truncated_full:
                break
            _final_step(T, U, V, lefts, kk, thin_u and build_uv, record)
        i += 1

    if truncated:
        out = {"Tk": np.asfortranarray(T[:k, :]), "V": V,
               "rho": float(np.linalg.norm(T[k:, k:]))}
        if build_uv:
            out["Uk"] = _thin_u(m, k, lefts) if thin_u else np.asfortranarray(U[:, :k])
        out["T"] = T
        return out
    out = {"T": T, "V": V}
    if build_uv:
        out["U"] = _thin_u(m, n, lefts) if thin_u else U
    return out


def _orth(X):
    """The first w columns of the Householder Q of X (h x w, h >= w):
    Q(:, 0:w) = (I - W T W^T) E = E - W (T W_1^T), E = [I_w; 0], W_1 = W[0:w, :]
    (dlarfg convention, oracle.householder)."""
    F, tau = householder_qr(X)
    W = unit_lower(F)
    Tq = larft(W, tau)
    w = X.shape[1]
    E = np.zeros_like(W)
    E[np.arange(w), np.arange(w)] = 1.0
    return np.asfortranarray(E - W @ (Tq @ W[:w, :].T))


def _sample(At, G, q, reorth=False):
    """O2: Y = (A_t^T A_t)^q A_t^T G, evaluated literally right to left (A8).
    reorth (NEXT-4): Y and Z are replaced by the orthonormal bases _orth(Y),
    _orth(Z) before each product -- the same column span in exact arithmetic
    (each _orth is a right multiplication by an invertible triangular factor),
    but directions below eps^(1/(2q+1)) of the top one survive (the standard
    power scheme of the randomized-SVD literature the paper cites)."""
    Y = At.T @ G
    for _ in range(q):
        if reorth:
            Y = _orth(Y)
        Z = At @ Y
        if reorth:
            Z = _orth(Z)
        Y = At.T @ Z
    return Y


def _select(At, Y, b):
    """Reading A28 (oversampling, NEXT-4): the sample Y has b + p columns
    (p <= s - b); keep
    the b directions of span(Y) along which A_t is largest -- the Rayleigh-Ritz
    choice of the randomized range finder the paper's construction comes from
    (P:651-656): Q_Y = _orth(Y); R_B = the R factor of B = A_t Q_Y (Householder,
    oracle.householder); R_B = U_R diag(d) V_R^T (oracle.jacobi.svd_block, d
    descending); return Y_hat = Q_Y V_R[:, 0:b], whose Householder QR then
    defines V_hat as without oversampling."""
    QY = _orth(Y)
    FB, _ = householder_qr(At @ QY)
    _, _, VR, _ = svd_block(upper_r(FB))
    return np.asfortranarray(QY @ VR[:, :b])


def _sampled_step(T, U, V, lefts, kk, b, q, seed, i, thin, record, reorth=False, oversample=0):
    m, n = T.shape
    r = m - kk
    # O1, O2 (with oversampling: b + p columns, the first b the same draws;
    # p capped at s - b, beyond which span(Y) cannot grow)
    p = min(oversample, (n - kk) - b)
    G = gaussian_block(seed, i, r, b + p)
    Y = _sample(T[kk:, kk:], G, q, reorth)
    if p > 0:
        Y = _select(T[kk:, kk:], Y, b)
    # O3, O4 on Y
    FY, tauV = householder_qr(Y)
    WV = unit_lower(FY)
    TV = larft(WV, tauV)
    # O5: right transform, all m rows of columns kk:n (A2); V likewise
    # (X -= ... is X := X - ... elementwise; in place only to hold one m x s
    # temporary at the full sizes)
    X = T[:, kk:]
    X -= _mm((X @ WV) @ TV, WV.T)
    if V is not None:
        XV = V[:, kk:]
        XV -= _mm((XV @ WV) @ TV, WV.T)
    # O6: left QR of the leading column block
    FU, tauU = householder_qr(T[kk:, kk:kk + b])
    WU = unit_lower(FU)
    TU = larft(WU, tauU)
    R = upper_r(FU)
    T[kk:kk + b, kk:kk + b] = R
    T[kk + b:, kk:kk + b] = 0.0
    # O7: left transform of the trailing columns (A3) and U
    Xl = T[kk:, kk + b:]
    Xl -= _mm(WU, TU.T @ (WU.T @ Xl))
    if U is not None:
        XU = U[:, kk:]
        XU -= _mm((XU @ WU) @ TU, WU.T)
    # O8, O9
    Us, d, Vs, sweeps = svd_block(R)
    _fold(T, U, V, kk, b, Us, d, Vs)
    if thin:
        lefts.append((kk, WU, TU, Us))
    if record is not None:
        record.setdefault("steps", []).append(
            {"i": i, "k": kk, "Y": Y, "tauV": tauV, "TV": TV, "tauU": tauU, "TU": TU,
             "R": R, "d": d, "sweeps": sweeps})


def _final_step(T, U, V, lefts, kk, thin, record):
    m, n = T.shape
    r, s = m - kk, n - kk
    WU = TU = None
    if r > s:
        FU, tauU = householder_qr(T[kk:, kk:])
        WU = unit_lower(FU)
        TU = larft(WU, tauU)
        R = upper_r(FU)
        T[kk:kk + s, kk:] = R
        T[kk + s:, kk:] = 0.0
        if U is not None:
            XU = U[:, kk:]
            U[:, kk:] = XU - _mm((XU @ WU) @ TU, WU.T)
        B = R
    else:
        B = np.array(T[kk:, kk:], order="F", copy=True)   # dense final block (O10)
    Us, d, Vs, sweeps = svd_block(B)
    _fold(T, U, V, kk, s, Us, d, Vs)
    if thin:
        lefts.append((kk, WU, TU, Us))
    if record is not None:
        record.setdefault("steps", []).append({"i": "final", "k": kk, "B": B, "d": d, "sweeps": sweeps})


def _fold(T, U, V, kk, w, Us, d, Vs):
    """O9: fold the SVD factors of the w x w diagonal block into T, U, V."""
    T[kk:kk + w, kk:kk + w] = np.diag(d)
    if kk > 0:
        T[:kk, kk:kk + w] = T[:kk, kk:kk + w] @ Vs
    if kk + w < T.shape[1]:
        T[kk:kk + w, kk + w:] = Us.T @ T[kk:kk + w, kk + w:]
    if U is not None:
        U[:, kk:kk + w] = U[:, kk:kk + w] @ Us
    if V is not None:
        V[:, kk:kk + w] = V[:, kk:kk + w] @ Vs


def _thin_u(m, c, lefts):
    """A12: U(:, :c) by backward accumulation of the recorded left transforms."""
    X = np.zeros((m, c), order="F")
    X[np.arange(c), np.arange(c)] = 1.0
    for kk, WU, TU, Us in reversed(lefts):
        w = Us.shape[0]
        if kk >= c:
            continue
        X[kk:kk + w, :] = Us @ X[kk:kk + w, :]
        if WU is not None:
            Xs = X[kk:, :]
            X[kk:, :] = Xs - _mm(WU, TU @ (WU.T @ Xs))
    return X


# ----------------------------------------------------------------------------
# Quantities derived from a factorisation (used by tests / bench checks)
# ----------------------------------------------------------------------------

def reconstruction_error(A, U, T, V):
    """||A - U T V^T||_F / ||A||_F."""
    nA = np.linalg.norm(A)
    R = A - (U[:, :T.shape[0]] @ T) @ V.T
    return float(np.linalg.norm(R) / (nA if nA > 0 else 1.0))


def orthogonality_error(Q):
    """||Q^T Q - I||_2 (spectral norm, reading A17)."""
    E = Q.T @ Q - np.eye(Q.shape[1])
    return float(np.linalg.norm(E, 2))

