"""The algorithmic flop models behind bench.py's GFLOP/s:
pinned to their closed-form asymptotics for n / b -> infinity."""
import pytest

from paper_2002_06960_b200.flops import hqrrp_flops, randutv_flops


@pytest.mark.parametrize("q", [0, 1, 2])
def test_randutv_flops_asymptotics(q):
    # square: (12 + 4q)/3 n^3 for T, + 4 n^3 for U and V (flops.py docstring)
    n, b = 65536, 64
    assert randutv_flops(n, n, b, q, build_uv=False) / n ** 3 == pytest.approx((12 + 4 * q) / 3, rel=5e-3)
    assert randutv_flops(n, n, b, q) / n ** 3 == pytest.approx((12 + 4 * q) / 3 + 4, rel=5e-3)


def test_hqrrp_flops_asymptotics():
    # sketch 2/3 n^3 + left updates 4/3 n^3 (+ Q: 2 n^3)
    n, b = 65536, 64
    assert hqrrp_flops(n, n, b, build_q=False) / n ** 3 == pytest.approx(2.0, rel=5e-3)
    assert hqrrp_flops(n, n, b) / n ** 3 == pytest.approx(4.0, rel=5e-3)


def test_truncated_flops_below_full():
    m, n, b, q = 262144, 8192, 256, 2
    assert randutv_flops(m, n, b, q, k=512) < randutv_flops(m, n, b, q)
