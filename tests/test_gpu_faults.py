"""Error paths under injected faults (RUTV_FAULT, SURVEY.md §5 "failure
detection"): a failed workspace allocation, the same on ONE rank of a sharded
call (the pre-collective agreement must return on every rank -- nobody left in
a collective), and a kernel failure in the middle of a factorisation (the
status comes back, the context stays usable).  Each case runs in a subprocess
(the injector reads its environment once) under a timeout, so a hang fails the
test instead of stalling the suite."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PRE = """
import sys, numpy as np, torch
sys.path.insert(0, %r)
sys.path.insert(0, %r)
from gpu_util import to_dev, to_np
from paper_2002_06960_b200 import randutv as r
""" % (ROOT, os.path.join(ROOT, "tests"))


def _run(code, fault, timeout=240):
    env = dict(os.environ, RUTV_FAULT=fault)
    p = subprocess.run([sys.executable, "-c", PRE + code], env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    return p.stdout


def test_fault_alloc_single_gpu():
    out = _run("""
c = r.Context()
A = to_dev(np.random.default_rng(0).standard_normal((200, 180)))
try:
    c.randutv_factor_ex(A, 32, 1, 3)
    print("NO ERROR")
except r.RandUTVError as e:
    assert e.status == r.RANDUTV_ERR_ALLOC, e.status
    assert "RUTV_FAULT" in c.lib.randutv_last_error().decode()
    print("ALLOC OK")
""", "alloc")
    assert "ALLOC OK" in out


def test_fault_alloc_one_rank_of_sharded_call():
    out = _run("""
A = np.random.default_rng(1).standard_normal((256, 192))
m, n, b = 256, 192, 32
locs = [to_dev(A[:, r.local_columns(n, b, 3, p)]) for p in range(3)]
try:
    r.randutv_factor_dist_loopback(locs, m, n, b, 1, 5)
    print("NO ERROR")
except r.RandUTVError as e:
    # rank 0 (first reported) saw its peer fail the agreement: RANDUTV_ERR_PEER
    assert e.status in (r.RANDUTV_ERR_PEER, r.RANDUTV_ERR_ALLOC), e.status
    print("AGREED", e.status == r.RANDUTV_ERR_PEER)
""", "alloc:rank=1", timeout=180)
    assert "AGREED True" in out


def test_fault_mid_factorisation_then_recovery():
    out = _run("""
A = np.random.default_rng(2).standard_normal((300, 260))
c = r.Context()
try:
    c.randutv_factor_ex(to_dev(A), 32, 1, 7)
    print("NO ERROR")
except r.RandUTVError as e:
    assert e.status == r.RANDUTV_ERR_CUDA, e.status
    print("FAILED AS INJECTED")
U, T, V, st = c.randutv_factor_ex(to_dev(A), 32, 1, 7)       # the same ctx: usable again
c2 = r.Context()
U2, T2, V2, _ = c2.randutv_factor_ex(to_dev(A), 32, 1, 7)    # a fresh ctx: the same bits
assert st == 0 and torch.equal(T, T2) and torch.equal(U, U2) and torch.equal(V, V2)
print("RECOVERED")
""", "launch:40")
    assert "FAILED AS INJECTED" in out and "RECOVERED" in out
