"""Host logic of the DGEMM work schedule (randutv_dgemm_plan, include/randutv.h;
DESIGN.md section 6: split-K and the tail-split of the last partial wave).  No GPU:
the planner is pure host arithmetic inside librandutv.so."""
import itertools

import pytest

from paper_2002_06960_b200.randutv import RandUTVError, randutv_dgemm_plan

SMS = 148
WS = 4 * 16384 * 256 + (1 << 17)  # the workspace randutv_dgemm itself hands over for a 16384 x 256 output


def _check_invariants(M, N, K, ws, p):
    gm, gn = -(-M // 64), -(-N // 64)
    assert p["tiles"] == gm * gn
    assert p["resident"] == 3 * SMS
    assert 0 <= p["full"] <= p["tiles"]
    tail = p["tiles"] - p["full"]
    if tail == 0:
        # unsplit: every tile whole, over all of K
        assert p["tsplits"] == 1 and p["partial_elems"] == 0
        assert p["kchunk"] == max(K, 1)
        return
    # whole-tile items fill complete waves (or there are none: plain split-K)
    assert p["full"] % p["resident"] == 0
    assert p["tsplits"] >= 2
    # the k-ranges are whole 32-wide k-tiles, at least 4 of them, and cover K exactly once
    assert p["kchunk"] % 32 == 0 and p["kchunk"] >= 128
    assert (p["tsplits"] - 1) * p["kchunk"] < K <= p["tsplits"] * p["kchunk"]
    # partial tiles fit the workspace
    assert p["partial_elems"] == tail * p["tsplits"] * 64 * 64 <= ws


@pytest.mark.parametrize("M,N,K", list(itertools.product([1, 63, 64, 300, 4096, 16384], [1, 256, 1000, 16128],
                                                         [0, 1, 31, 512, 3072, 6144, 16384, 262144])))
def test_plan_invariants(M, N, K):
    for ws in (0, 1 << 16, WS, 1 << 30):
        for tail in (True, False):
            _check_invariants(M, N, K, ws, randutv_dgemm_plan(M, N, K, ws, SMS, tail))


def test_no_workspace_never_splits():
    p = randutv_dgemm_plan(64, 48, 20000, 0, SMS)
    assert p["full"] == p["tiles"] == 1 and p["tsplits"] == 1 and p["kchunk"] == 20000


def test_skinny_long_k_splits_every_tile():
    # S2 of c4: 256 x 8192^T... here the 64 x 48 x 20000 test shape: one tile, split over the chip
    p = randutv_dgemm_plan(64, 48, 20000, 1 << 20, SMS)
    assert p["full"] == 0 and p["tsplits"] > 8


def test_tail_split_on_the_c3_late_skinny_products():
    # X W_V at c3 step 48 (16384 x 256 x 4096): 1024 tiles on 444 slots = 2.3 waves;
    # the two full waves stay whole, the 136-tile tail is split (profiles/gemm_tail_r02d.txt)
    p = randutv_dgemm_plan(16384, 256, 4096, WS, SMS)
    assert p["tiles"] == 1024 and p["full"] == 888 and p["tsplits"] >= 2
    # the switch leaves only the unsplit and plain split-K schedules
    q = randutv_dgemm_plan(16384, 256, 4096, WS, SMS, tail_split=False)
    assert q["full"] in (0, q["tiles"])


def test_tail_split_gated_off_for_long_k():
    # measured slower on long-K products (K > 6144): their whole-tile items straggle
    p = randutv_dgemm_plan(16384, 256, 16384, WS, SMS)
    assert p["full"] in (0, p["tiles"])


def test_big_outputs_stay_unsplit():
    # the fused rank-2b update of c3 step 0: 64512 tiles = 145.3 waves, a tail split gains < 3 %
    p = randutv_dgemm_plan(16384, 16128, 512, 1 << 28, SMS)
    assert p["full"] == p["tiles"] and p["tsplits"] == 1


def test_argument_errors():
    for bad, idx in (((-1, 1, 1, 0, SMS), 1), ((1, -1, 1, 0, SMS), 2), ((1, 1, -1, 0, SMS), 3),
                     ((1, 1, 1, -1, SMS), 4), ((1, 1, 1, 0, 0), 5)):
        with pytest.raises(RandUTVError) as e:
            randutv_dgemm_plan(*bad)
        assert f"-{idx}" in str(e.value) or getattr(e.value, "status", None) == -idx


def test_empty_output():
    p = randutv_dgemm_plan(0, 5, 7, 100, SMS)
    assert p["tiles"] == 0 and p["full"] == 0 and p["partial_elems"] == 0
