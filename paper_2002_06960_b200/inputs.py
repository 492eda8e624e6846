"""Seeded synthetic input matrices for the configs of BASELINE.json.

This module holds NO randUTV arithmetic: it only builds the matrices A that both
the CUDA path and the CPU oracle factor (the paper's workloads are "randomly
generated" FP64 matrices).  Both sides receive the same bytes.

Recipes (SURVEY.md §8(d) M2 and readings A18-A20):
  c1  n=512:   A = U0 diag(10^(-8(i-1)/(n-1))) V0^T, U0, V0 Haar (QR of N(0,1)
               with the Mezzadri sign fix, A20)
  c2  n=4096:  A = N(0,1)^{n x n}
  c3  n=16384: A = U0 diag(exp(-(i-1)/1000)) V0^T + 1e-12 E, E = N(0,1)   (A18)
  c4  262144 x 8192: A = X diag(10^(-3(j-1)/499)) Y^T + 1e-6 E, X, Y orthonormal
               m x 500 / n x 500 (thin QR of N(0,1), sign fix), E = N(0,1)   (A19)
  c5  n=65536: A = N(0,1)^{n x n}
Seeds: seed_A = 1000+c, seed_U0 = 4000+c, seed_V0 = 5000+c, seed_E = 3000+c,
seed_G = 2000+c for config c.

Two back ends build the same recipe: numpy (host, PCG64 streams; used by the
CPU tests and the oracle parity tests) and torch on a CUDA device (Philox
streams of torch; used for the multi-GB bench inputs, where a host QR of a
16384^2 matrix would dominate the run).  They give different bytes for the same
seed, so a test always hands one generated array to both sides.
"""
import numpy as np

CONFIGS = {
    "c1": dict(m=512, n=512, b=64, q=2, kind="powspec", full=True, ks=(64, 128)),
    "c2": dict(m=4096, n=4096, b=128, q=1, kind="gauss", full=True),
    "c3": dict(m=16384, n=16384, b=256, q=2, kind="expspec", full=True),
    "c4": dict(m=262144, n=8192, b=256, q=2, kind="lowrank", full=False, k=512),
    "c5": dict(m=65536, n=65536, b=512, q=1, kind="gauss", full=True),
}


def seeds(cfg_index):
    c = int(cfg_index)
    return dict(A=1000 + c, E=3000 + c, U0=4000 + c, V0=5000 + c, G=2000 + c)


# --------------------------------------------------------------------------- numpy

def _rng(seed):
    return np.random.default_rng(int(seed))


def gaussian(m, n, seed):
    return np.asfortranarray(_rng(seed).standard_normal((m, n)))


def haar(n, seed, cols=None):
    """Haar-distributed orthogonal n x n (or n x cols orthonormal) matrix (A20)."""
    c = n if cols is None else cols
    Z = _rng(seed).standard_normal((n, c))
    Q, R = np.linalg.qr(Z)
    sgn = np.sign(np.diag(R))
    sgn[sgn == 0] = 1.0
    return np.asfortranarray(Q * sgn)


def known_spectrum(sigma, seed_u, seed_v, m=None):
    n = len(sigma)
    m = n if m is None else m
    U0 = haar(m, seed_u, cols=n)
    V0 = haar(n, seed_v)
    return np.asfortranarray((U0 * np.asarray(sigma)) @ V0.T)


def sigma_powspec(n, decades=8.0):
    i = np.arange(n, dtype=np.float64)
    return 10.0 ** (-decades * i / max(n - 1, 1))


def sigma_expspec(n, scale=1000.0):
    return np.exp(-np.arange(n, dtype=np.float64) / scale)


def make_numpy(kind, m, n, cfg_index=0, noise=None, rank=None):
    """Build a config-shaped matrix on the host with numpy."""
    sd = seeds(cfg_index)
    if kind == "gauss":
        return gaussian(m, n, sd["A"])
    if kind == "powspec":
        return known_spectrum(sigma_powspec(n), sd["U0"], sd["V0"], m=m)
    if kind == "expspec":
        A = known_spectrum(sigma_expspec(n), sd["U0"], sd["V0"], m=m)
        return np.asfortranarray(A + (1e-12 if noise is None else noise) * gaussian(m, n, sd["E"]))
    if kind == "lowrank":
        k = 500 if rank is None else rank
        X = haar(m, sd["U0"], cols=k)
        Y = haar(n, sd["V0"], cols=k)
        s = 10.0 ** (-3.0 * np.arange(k) / max(k - 1, 1))
        A = (X * s) @ Y.T
        return np.asfortranarray(A + (1e-6 if noise is None else noise) * gaussian(m, n, sd["E"]))
    raise ValueError(kind)


def make_config_numpy(name):
    c = CONFIGS[name]
    return make_numpy(c["kind"], c["m"], c["n"], cfg_index=int(name[1:]))


# --------------------------------------------------------------------------- torch (GPU)

def make_torch(kind, m, n, cfg_index=0, device="cuda", noise=None, rank=None):
    """Same recipes built with torch on `device`; returns a column-major float64
    tensor, i.e. an (n, m) row-major tensor whose transpose view is A."""
    import torch

    sd = seeds(cfg_index)

    def g(seed, r, c):
        gen = torch.Generator(device=device)
        gen.manual_seed(int(seed))
        return torch.randn((r, c), generator=gen, device=device, dtype=torch.float64)

    def haar_t(seed, r, c):
        Q, R = torch.linalg.qr(g(seed, r, c))
        sgn = torch.sign(torch.diagonal(R))
        sgn[sgn == 0] = 1.0
        return Q * sgn

    if kind == "gauss":
        A = g(sd["A"], n, m).t()          # column-major m x n
    elif kind in ("powspec", "expspec"):
        sig = torch.arange(n, device=device, dtype=torch.float64)
        sig = 10.0 ** (-8.0 * sig / max(n - 1, 1)) if kind == "powspec" else torch.exp(-sig / 1000.0)
        U0 = haar_t(sd["U0"], m, n)
        V0 = haar_t(sd["V0"], n, n)
        At = (V0 * sig) @ U0.t()          # = A^T, row-major (n, m) == A column-major
        del U0, V0
        if kind == "expspec":
            At.add_(g(sd["E"], n, m), alpha=(1e-12 if noise is None else noise))
        A = At.t()
    elif kind == "lowrank":
        k = 500 if rank is None else rank
        X = haar_t(sd["U0"], m, k)
        Y = haar_t(sd["V0"], n, k)
        s = 10.0 ** (-3.0 * torch.arange(k, device=device, dtype=torch.float64) / max(k - 1, 1))
        At = (Y * s) @ X.t()
        del X, Y
        At.add_(g(sd["E"], n, m), alpha=(1e-6 if noise is None else noise))
        A = At.t()
    else:
        raise ValueError(kind)
    assert A.stride(0) == 1 and A.stride(1) == m
    return A


def make_config_torch(name, device="cuda"):
    c = CONFIGS[name]
    return make_torch(c["kind"], c["m"], c["n"], cfg_index=int(name[1:]), device=device)
