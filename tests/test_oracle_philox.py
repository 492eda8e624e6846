"""Pins for oracle O1 (the Gaussian G, reading A7)."""
import os

import numpy as np
import pytest
from scipy import stats

from oracle.philox import gaussian_block, philox4x32_10

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        lhs, rhs = line.split("->")
        rows.append(([int(x, 16) for x in lhs.split()], [int(x, 16) for x in rhs.split()]))
    return rows


@pytest.mark.parametrize("case", _kat())
def test_philox_known_answers(case):
    (c0, c1, c2, c3, k0, k1), expect = case
    out = philox4x32_10(c0, c1, c2, c3, k0, k1)
    assert [int(o) for o in out] == expect


def test_gaussian_moments():
    # 10^6 samples: mean within 0.01, variance within 0.02, plus
    # third/fourth moments of N(0,1) (0 and 3), which a wrong Box-Muller branch breaks.
    g = gaussian_block(12345, 0, 2000, 500).ravel()
    assert abs(g.mean()) < 0.01
    assert abs(g.var() - 1.0) < 0.02
    assert abs(stats.skew(g)) < 0.02
    assert abs(stats.kurtosis(g, fisher=False) - 3.0) < 0.05


def test_gaussian_ks_even_odd_rows_and_independence():
    g = gaussian_block(7, 3, 4000, 50)
    even, odd = g[0::2].ravel(), g[1::2].ravel()
    assert stats.kstest(even, "norm").pvalue > 1e-3
    assert stats.kstest(odd, "norm").pvalue > 1e-3
    # cos/sin branches of one Philox draw are independent N(0,1): correlation ~ 0
    assert abs(np.corrcoef(even, odd)[0, 1]) < 0.02


def test_gaussian_order_independent_and_keyed():
    full = gaussian_block(99, 5, 301, 17)
    part = gaussian_block(99, 5, 100, 17, row0=151)
    assert np.array_equal(full[151:251], part)
    assert np.array_equal(full, gaussian_block(99, 5, 301, 17))
    assert not np.array_equal(full, gaussian_block(99, 6, 301, 17))
    assert not np.array_equal(full, gaussian_block(100, 5, 301, 17))
    # the high half of a 64-bit seed is part of the key
    assert not np.array_equal(gaussian_block(1, 0, 8, 4), gaussian_block(1 + (1 << 32), 0, 8, 4))
    assert full.flags.f_contiguous
