"""Helpers for the -m gpu parity tests (test-side verification only)."""
import numpy as np

U64 = 2.0 ** -53


def to_np(X):
    """Column-major device tensor -> Fortran numpy array."""
    return np.asfortranarray(X.detach().cpu().numpy())


def to_dev(A, device="cuda"):
    """Fortran numpy array -> column-major device tensor (strides (1, m))."""
    import torch
    A = np.asfortranarray(A, dtype=np.float64)
    m, n = A.shape
    t = torch.empty((n, m), dtype=torch.float64, device=device)
    t.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
    return t.t()


def diag_parity(d_gpu, d_ora):
    """Reading A16: |Delta_k| <= 1e-9 |T_o(k,k)| + 1e-14 |T_o(1,1)|; returns the max ratio to the bound."""
    a, o = np.abs(d_gpu), np.abs(d_ora)
    bound = 1e-9 * o + 1e-14 * o.max()
    return float(np.max(np.abs(a - o) / bound))


def spectral_orth_error(Q):
    """||Q^T Q - I||_2 on the host (exact, via LAPACK eigvalsh)."""
    E = Q.T @ Q - np.eye(Q.shape[1])
    return float(np.max(np.abs(np.linalg.eigvalsh(E))))


def recon_error(A, U, T, V):
    return float(np.linalg.norm(A - (U[:, :T.shape[0]] @ T) @ V.T) / max(np.linalg.norm(A), 1e-300))
