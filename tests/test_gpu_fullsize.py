"""Parity and invariants at BASELINE.json's FULL sizes, in the launch
configuration bench.py times (one ctx on cuda:0, the configs' b, q and seeds,
inputs generated on the GPU by paper_2002_06960_b200.inputs).

The oracle cannot factor these matrices whole, so (test plan):
  * sampled outputs the oracle computes directly: the first sampled step of
    c3 (truncated k = b: T(0:b, :), U(:, 0:b), rho) on the same A bytes;
  * properties that hold at any size, evaluated on the GPU with torch
    (cuBLAS / cuSOLVER FP64, test-side only): reconstruction, orthogonality,
    exact triangularity, ||T||_F = ||A||_F, |det A| = prod |T_kk| (LU), and
    for the truncated c4 run the exact optimum sigma_{k+1..n} of A (QR + SVD)
    bounding ||A - A_k||_F from below.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import diag_parity  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    from paper_2002_06960_b200.randutv import Context
    c = Context()
    yield c
    c.close()


def _orth_err_exact(Q):
    import torch
    E = Q.t() @ Q
    E.diagonal().sub_(1.0)
    return float(torch.linalg.eigvalsh(E).abs().max())


def _orth_err_power(Q, iters=40, block=8, seed=0):
    """||Q^T Q - I||_2 by block power iteration on the implicit symmetric E
    (too large to form at n = 65536): converges to the extreme eigenvalue."""
    import torch
    g = torch.Generator(device=Q.device)
    g.manual_seed(seed)
    X = torch.randn((Q.shape[1], block), generator=g, device=Q.device, dtype=torch.float64)
    est = 0.0
    for _ in range(iters):
        X, _ = torch.linalg.qr(X)
        Y = Q.t() @ (Q @ X) - X
        est = float(torch.linalg.matrix_norm(Y, 2))
        X = Y
    return est


def _logabsdet(A):
    import torch
    # det A^T = det A; A^T of a column-major A is a contiguous row-major tensor (no copy)
    return float(torch.linalg.slogdet(A.t())[1])


def test_c3_fullsize(ctx):
    import torch
    from oracle.randutv import randutv as oracle_randutv
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    c = CONFIGS["c3"]
    m, n, b, q, seed = c["m"], c["n"], c["b"], c["q"], 2003
    A = make_config_torch("c3")
    nA = float(torch.linalg.norm(A))
    lad = _logabsdet(A)
    U, T, V, st = ctx.randutv_factor_ex(A, b, q, seed)
    assert st == 0
    R = A - (U @ T) @ V.t()
    assert float(torch.linalg.norm(R)) / nA <= 1e-12
    del R
    assert _orth_err_exact(U) <= 1e-12
    assert _orth_err_exact(V) <= 1e-12
    assert bool((torch.tril(T, -1) == 0).all())
    assert abs(float(torch.linalg.norm(T)) - nA) <= 1e-13 * nA * 10
    d = torch.diagonal(T).abs()
    assert abs(float(torch.log(d).sum()) - lad) <= 1e-5
    # sampled oracle parity: the first sampled step on the same bytes
    Uk, Tk, Vk, rho = ctx.randutv_factor_rank(A, b, b, q, seed)
    Ah = np.asfortranarray(A.cpu().numpy())
    o = oracle_randutv(Ah, b, q, seed, k=b, thin_u=True)
    Tk = Tk.cpu().numpy()
    assert np.max(np.abs(np.abs(Tk) - np.abs(o["Tk"]))) / nA <= 1e-11
    assert diag_parity(np.diag(Tk[:, :b]), np.diag(o["Tk"][:, :b])) <= 1.0
    assert abs(rho - o["rho"]) <= 1e-9 * o["rho"]
    assert np.max(np.abs(np.abs(Uk.cpu().numpy()) - np.abs(o["Uk"]))) <= 1e-9
    # the full run's first diagonal block is the truncated run's
    assert diag_parity(d[:b].cpu().numpy(), np.diag(o["Tk"][:, :b])) <= 1.0


def test_c4_fullsize_truncated(ctx):
    import torch
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    c = CONFIGS["c4"]
    m, n, b, q, k, seed = c["m"], c["n"], c["b"], c["q"], c["k"], 2004
    A = make_config_torch("c4")
    nA = float(torch.linalg.norm(A))
    Uk, Tk, V, rho = ctx.randutv_factor_rank(A, k, b, q, seed)
    # rho == ||A - Uk Tk V^T||_F (T(k:m, 0:k) = 0 exactly)
    Ak = Uk @ (Tk @ V.t())
    assert abs(float(torch.linalg.norm(A - Ak)) - rho) <= 1e-12 * nA
    del Ak
    assert _orth_err_exact(Uk) <= 1e-12
    assert _orth_err_exact(V) <= 1e-12
    assert bool((torch.tril(Tk[:, :k], -1) == 0).all())
    # exact singular values of A (QR, then SVD of the n x n R)
    Rf = torch.linalg.qr(A, mode="r")[1]
    sv = torch.linalg.svdvals(Rf)
    del Rf
    opt = float(torch.sqrt((sv[k:] ** 2).sum()))
    # Eckart-Young: no rank-k approximation beats sigma_{k+1..n}; q = 2 power
    # iteration comes within a few percent (calibrated, SURVEY.md §8(c) c4 pins)
    assert opt * (1 - 1e-12) <= rho <= 1.05 * opt
    # noise edge: 1e-6 (sqrt(m) + sqrt(n)) ~ 6e-4 bounds sigma_{k+1}
    assert float(sv[k]) <= 1e-6 * (math.sqrt(m) + math.sqrt(n)) * 1.05
    # the signal singular values are revealed on the diagonal of T
    dk = torch.diagonal(Tk[:, :k]).abs()
    rel = (dk[:500] / sv[:500] - 1).abs()
    assert float(rel.median()) <= 1e-2


def test_c5_fullsize(ctx):
    import torch
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    from paper_2002_06960_b200.randutv import colmajor
    c = CONFIGS["c5"]
    m, n, b, q, seed = c["m"], c["n"], c["b"], c["q"], 2005
    A = make_config_torch("c5")
    nA = float(torch.linalg.norm(A))
    lad = _logabsdet(A)
    torch.cuda.empty_cache()
    T = colmajor(m, n)
    U, T, V, st = ctx.randutv_factor_ex(A, b, q, seed, T=T)
    assert st == 0
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    X = torch.randn((n, 8), generator=g, device="cuda", dtype=torch.float64)
    Y1 = A @ X
    Y2 = U @ (T @ (V.t() @ X))
    assert float(torch.linalg.norm(Y1 - Y2) / torch.linalg.norm(Y1)) <= 1e-12
    del Y1, Y2
    assert _orth_err_power(U) <= 1e-12
    assert _orth_err_power(V) <= 1e-12
    del U, V
    torch.cuda.empty_cache()
    for c0 in range(0, n, 4096):  # strict lower part exactly zero (in column chunks: no 32 GB temporary)
        assert bool((torch.tril(T[:, c0:c0 + 4096], -1 - c0) == 0).all())
    assert abs(float(torch.linalg.norm(T)) - nA) <= 1e-12 * nA
    d = torch.diagonal(T).abs()
    assert abs(float(torch.log(d).sum()) - lad) <= 1e-4


def test_c3_fullsize_hqrrp(ctx):
    """HQRRP on c3's full matrix: A P = Q R, Q orthogonal,
    R exactly upper triangular; the first block's pivots (a sketch CPQR over
    all 16384 columns) and the partial run's rho against the oracle on the
    same bytes."""
    import torch
    from oracle.hqrrp import hqrrp as oracle_hqrrp
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    from paper_2002_06960_b200.randutv import colmajor
    c = CONFIGS["c3"]
    b, seed = c["b"], 2003
    A = make_config_torch("c3")
    nA = float(torch.linalg.norm(A))
    R = colmajor(*A.shape)
    R.copy_(A)
    Q, jp = ctx.randutv_hqrrp(R, b, seed)
    torch.cuda.synchronize()
    assert bool((torch.sort(jp).values == torch.arange(A.shape[1], device=jp.device)).all())
    E = A.index_select(1, jp) - Q @ R
    assert float(torch.linalg.norm(E)) / nA <= 1e-12
    del E
    assert _orth_err_exact(Q) <= 1e-12
    assert bool((torch.tril(R, -1) == 0).all())
    del Q
    # the first block against the oracle (partial run, k = b)
    R.copy_(A)
    _, jpk, rho = ctx.randutv_hqrrp_rank(R, b, b, seed, build_q=False)
    Ah = np.asfortranarray(A.cpu().numpy())
    _, Ro, jpo, rho_o = oracle_hqrrp(Ah, b, seed, build_q=False, k=b)
    assert np.array_equal(jp[:b].cpu().numpy(), jpo[:b])
    assert np.array_equal(jpk.cpu().numpy(), jpo)
    assert abs(rho - rho_o) <= 1e-9 * rho_o
    assert np.max(np.abs(R[:b, :].cpu().numpy() - Ro[:b, :])) / nA <= 1e-11
