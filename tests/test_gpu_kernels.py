"""GPU parity of the individual steps (through the C ABI) against the oracle.

S1 Gaussian vs oracle.philox; S2/S3/S5/S7 DMMA GEMM vs an FP64 reference with
the componentwise GEMM error bound; S4/S6 panel QR vs oracle.householder;
S8 Jacobi SVD vs LAPACK singular values and the oracle's invariants.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import U64, to_dev, to_np  # noqa: E402
from oracle.householder import householder_qr, larft, unit_lower  # noqa: E402
from oracle.philox import gaussian_block  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device"
    from paper_2002_06960_b200.randutv import Context
    c = Context()
    yield c
    c.close()


# ------------------------------------------------------------------------- S1
@pytest.mark.parametrize("seed,it,rows,cols", [(2001, 0, 512, 64), (7, 3, 1001, 33), (2**40 + 5, 17, 1, 1),
                                               (123, 1, 65537, 8)])
def test_gaussian_matches_oracle(ctx, seed, it, rows, cols):
    G = to_np(ctx.randutv_gaussian(seed, it, rows, cols))
    Go = gaussian_block(seed, it, rows, cols)
    # same Philox bits; CUDA vs glibc log/sincos differ by a few ulps
    assert np.max(np.abs(G - Go) / np.maximum(1.0, np.abs(Go))) <= 16 * U64


# ------------------------------------------------------------------------- K2 GEMM
GEMM_CASES = [
    (0, 0, 300, 200, 100), (1, 0, 257, 129, 1000), (0, 1, 128, 128, 64), (1, 1, 65, 191, 33),
    (1, 0, 64, 48, 20000),   # split-K path
    (0, 0, 5000, 64, 4096), (0, 1, 1000, 1000, 256), (1, 0, 3, 1, 7), (0, 0, 1, 1, 1),
    # tail-split schedule (whole tiles for the full waves of 444 slots, the
    # last partial wave split into k-ranges + tail_reduce_kernel), ragged edges
    (0, 0, 8000, 250, 2100), (1, 0, 7001, 300, 3001), (0, 1, 8192, 256, 2048),
]


@pytest.mark.parametrize("ta,tb,M,N,K", GEMM_CASES)
@pytest.mark.parametrize("offset", [0, 1])
def test_dgemm_componentwise_bound(ctx, ta, tb, M, N, K, offset):
    import torch
    rng = np.random.default_rng(M + N + K + offset)
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    # offset = 1: odd leading dimensions and 8-byte-aligned (not 16) base pointers
    Abig = rng.standard_normal((ar + offset, ac + 1))
    Bbig = rng.standard_normal((br + offset, bc + 1))
    Cbig = rng.standard_normal((M + offset, N + 1))
    Ad, Bd, Cd = to_dev(Abig), to_dev(Bbig), to_dev(Cbig)
    A = Ad[offset:offset + ar, 1:1 + ac]
    B = Bd[offset:offset + br, 1:1 + bc]
    C = Cd[offset:offset + M, 1:1 + N]
    alpha, beta = -1.25, 0.5
    An = Abig[offset:offset + ar, 1:1 + ac]
    Bn = Bbig[offset:offset + br, 1:1 + bc]
    Cn = Cbig[offset:offset + M, 1:1 + N]
    ctx.randutv_dgemm(ta, tb, A, B, C, alpha=alpha, beta=beta)
    opA = An.T if ta else An
    opB = Bn.T if tb else Bn
    ref = alpha * (opA @ opB) + beta * Cn
    bound = (K + 2) * U64 * (abs(alpha) * (np.abs(opA) @ np.abs(opB)) + abs(beta) * np.abs(Cn)) * 2
    got = to_np(Cd)[offset:offset + M, 1:1 + N]
    assert np.all(np.abs(got - ref) <= bound + 1e-300)
    # the elements outside the view are untouched
    full = to_np(Cd)
    mask = np.ones_like(full, dtype=bool)
    mask[offset:offset + M, 1:1 + N] = False
    assert np.array_equal(full[mask], Cbig[mask])
    torch.cuda.synchronize()


def test_dgemm_beta_zero_ignores_nan(ctx):
    import torch
    rng = np.random.default_rng(3)
    A = to_dev(rng.standard_normal((70, 40)))
    B = to_dev(rng.standard_normal((40, 90)))
    C = to_dev(np.full((70, 90), np.nan))
    ctx.randutv_dgemm(0, 0, A, B, C, beta=0.0)
    assert torch.isfinite(C).all()


# ------------------------------------------------------------------------- S4/S6 QR
# (cluster leaf variants of qr.cu's leaf_plan: slab <= 4096 rows R=1; <= 8192 R=2;
#  <= 12288, 16384, 20480 R=2 plus 1, 2, 3 rows per thread in shared memory)
@pytest.mark.parametrize("h,w", [(1000, 64), (777, 45), (300, 300), (5000, 128), (40, 1), (33, 32), (4096, 256),
                                 (10000, 64), (16384, 96), (20000, 64), (20513, 40)])
def test_panel_qr_matches_oracle(ctx, h, w):
    rng = np.random.default_rng(h * 7 + w)
    P = rng.standard_normal((h, w))
    Pd = to_dev(P)
    _, tau, Tf = ctx.randutv_panel_qr(Pd)
    F = to_np(Pd)
    Fo, tauo = householder_qr(P)
    Wo = unit_lower(Fo)
    To = larft(Wo, tauo)
    kappa = np.linalg.cond(P)
    tol = 20 * kappa * h * U64
    assert np.max(np.abs(tau.cpu().numpy() - tauo)) <= tol
    assert np.max(np.abs(np.triu(F[:w]) - np.triu(Fo[:w]))) <= tol * np.linalg.norm(P)
    assert np.max(np.abs(np.tril(F, -1) - np.tril(Fo, -1))) <= tol
    assert np.max(np.abs(to_np(Tf) - To)) <= tol * max(1.0, np.max(np.abs(To)))
    assert np.all(np.tril(to_np(Tf), -1) == 0.0)


def test_panel_qr_deterministic(ctx):
    rng = np.random.default_rng(5)
    P = rng.standard_normal((3000, 96))
    outs = []
    for _ in range(2):
        Pd = to_dev(P)
        _, tau, Tf = ctx.randutv_panel_qr(Pd)
        outs.append((to_np(Pd), tau.cpu().numpy(), to_np(Tf)))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_panel_qr_identity_and_zero_columns(ctx):
    P = np.zeros((50, 4))
    P[:4, :4] = np.eye(4)
    Pd = to_dev(P)
    _, tau, Tf = ctx.randutv_panel_qr(Pd)
    assert np.all(tau.cpu().numpy() == 0.0)
    assert np.array_equal(to_np(Pd), P)


# ------------------------------------------------------------------------- S8 SVD
@pytest.mark.parametrize("w,kind", [(1, "dense"), (2, "dense"), (7, "dense"), (64, "tri"), (100, "dense"),
                                    (128, "graded"), (256, "tri"), (255, "dense"), (512, "tri"), (512, "graded")])
def test_small_svd_matches_lapack(ctx, w, kind):
    # "tri": the R factor of a Gaussian matrix (what S6 hands to S8 on a Gaussian A);
    # "graded": R of U0 diag(10^(-8 i/w)) V0^T (a c1-like block with 8 decades)
    rng = np.random.default_rng(w)
    B = rng.standard_normal((w, w))
    if kind == "tri":
        B = np.linalg.qr(B)[1]
    elif kind == "graded":
        Q1 = np.linalg.qr(rng.standard_normal((w, w)))[0]
        Q2 = np.linalg.qr(rng.standard_normal((w, w)))[0]
        B = np.linalg.qr((Q1 * 10.0 ** (-8.0 * np.arange(w) / w)) @ Q2.T)[1]
    Us, d, Vs, st = ctx.randutv_small_svd(to_dev(B))
    Us, d, Vs = to_np(Us), d.cpu().numpy(), to_np(Vs)
    s = np.linalg.svd(B, compute_uv=False)
    assert np.all(np.diff(d) <= 0) and np.all(d >= 0)
    assert np.max(np.abs(d - s)) <= 10 * w * U64 * s[0]
    assert np.linalg.norm(B - (Us * d) @ Vs.T) <= 1e-13 * np.linalg.norm(B) * max(1, w / 64)
    assert np.linalg.norm(Us.T @ Us - np.eye(w), 2) <= 1e-13 * max(1, w / 64)
    assert np.linalg.norm(Vs.T @ Vs - np.eye(w), 2) <= 1e-13 * max(1, w / 64)


def test_small_svd_golden_cases(ctx):
    # tests/golden/small_cases.txt: svd_diag, svd_zero
    Us, d, Vs, _ = ctx.randutv_small_svd(to_dev(np.diag([3.0, 1.0, 2.0])))
    assert np.array_equal(d.cpu().numpy(), [3.0, 2.0, 1.0])
    P = np.eye(3)[:, [0, 2, 1]]
    assert np.array_equal(np.abs(to_np(Us)), P) and np.array_equal(np.abs(to_np(Vs)), P)
    Us, d, Vs, _ = ctx.randutv_small_svd(to_dev(np.zeros((3, 3))))
    assert np.array_equal(d.cpu().numpy(), [0.0, 0.0, 0.0])
    assert np.array_equal(to_np(Us), np.eye(3)) and np.array_equal(to_np(Vs), np.eye(3))


def test_small_svd_rank_deficient_completion(ctx):
    rng = np.random.default_rng(9)
    B = np.zeros((6, 6))
    B[:, 1] = rng.standard_normal(6)
    B[:, 4] = rng.standard_normal(6)
    Us, d, Vs, _ = ctx.randutv_small_svd(to_dev(B))
    Us, d, Vs = to_np(Us), d.cpu().numpy(), to_np(Vs)
    assert np.count_nonzero(d) == 2
    assert np.linalg.norm(Us.T @ Us - np.eye(6)) < 1e-14
    assert np.linalg.norm(B - (Us * d) @ Vs.T) < 1e-14 * np.linalg.norm(B)
