"""O1 -- the Gaussian test matrix G^(i) (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Paper: "Draw a random matrix G^(i) in R^{(m-ib) x b}, with i.i.d. entries drawn
from the standard normal distribution" (Sec. 3.1, construction of
V-hat step 1); FLAME form ``G := generate_iid_stdnorm_matrix(m(A) - m(A00), n_b)``
(Fig. fig:FLArandutv).  The paper does not name a generator
(reading A7), so both sides implement the same counter-based one:

* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), multipliers
  0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85.
* entry (row, col) of G^(i):  counter = (row >> 1, col, i, 0),
  key = (seed mod 2^32, seed >> 32)  ->  (o0, o1, o2, o3)
* u1 = ((o0<<32 | o1) >> 11) * 2^-53 + 2^-54     in (0, 1)
  u2 = ((o2<<32 | o3) >> 11) * 2^-53             in [0, 1)
* Box-Muller: rho = sqrt(-2 ln u1), theta = 2*pi*u2;
  G = rho*cos(theta) for even row, rho*sin(theta) for odd row.

Rows are numbered in the trailing coordinates of iteration i (reading A6:
G has m - k rows, k = i*b, as FLAME's ``m(A) - m(A00)``).
"""
import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds, elementwise over broadcastable uint32 inputs.

    Round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2 (64-bit products);
    c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by the
    Weyl constants before every round after the first.
    Returns four uint64 arrays holding 32-bit values.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0 = _M0 * c0          # < 2^64: exact in uint64
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def uniforms_from_bits(o0, o1, o2, o3):
    """(u1, u2) from one Philox output block, as stated in the module docstring."""
    w1 = (o0 << _S32) | o1
    w2 = (o2 << _S32) | o3
    u1 = (w1 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 + 2.0 ** -54
    u2 = (w2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return u1, u2


def gaussian_block(seed, it, rows, cols, row0=0):
    """G^(it)[row0:row0+rows, 0:cols] as a column-major (Fortran) float64 array."""
    seed = int(seed)
    r = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    c = np.arange(cols, dtype=np.uint64)[None, :]
    o0, o1, o2, o3 = philox4x32_10(r >> np.uint64(1), c, np.uint64(it), np.uint64(0),
                                   seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    u1, u2 = uniforms_from_bits(o0, o1, o2, o3)
    rho = np.sqrt(-2.0 * np.log(u1))
    theta = 6.283185307179586 * u2
    even = (r & np.uint64(1)) == 0
    g = np.where(even, rho * np.cos(theta), rho * np.sin(theta))
    return np.asfortranarray(g)
