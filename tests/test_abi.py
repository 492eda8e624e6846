"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/randutv.h declares (no compute calls: there may be no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "randutv.h")


def _declared():
    src = open(HEADER).read()
    return re.findall(r"RANDUTV_API\s+[\w\s\*]+?\b(randutv_\w+)\s*\(", src)


@pytest.fixture(scope="module")
def lib():
    from paper_2002_06960_b200 import build as b
    b.build()
    from paper_2002_06960_b200.randutv import load_library
    return load_library()


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("randutv_factor", "randutv_factor_ex", "randutv_factor_rank", "randutv_create",
                     "randutv_destroy", "randutv_gaussian", "randutv_dgemm", "randutv_panel_qr",
                     "randutv_small_svd"):
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2002_06960_b200.randutv import SIGNATURES
    names = _declared()
    assert len(names) == len(set(names))
    for name in names:
        assert hasattr(lib, name), name
    # the binding covers exactly the declared symbols
    assert set(SIGNATURES) == set(names)


def test_only_the_abi_is_exported():
    import subprocess
    so = os.path.join(ROOT, "paper_2002_06960_b200", "librandutv.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(_declared())


def test_host_only_entries(lib):
    out = ctypes.c_size_t()
    assert lib.randutv_workspace_bytes(4096, 4096, 128, 1, 0, ctypes.byref(out)) == 0
    assert out.value > 4096 * 128 * 8 * 6
    assert lib.randutv_workspace_bytes(10, 20, 4, 1, 0, ctypes.byref(out)) == -1
    assert lib.randutv_workspace_bytes(10, 10, 0, 1, 0, ctypes.byref(out)) == -3
    assert b"success" in lib.randutv_status_string(0)
    assert lib.randutv_destroy(None) == 0x40000003


def test_status_codes_do_not_collide(lib):
    """Jacobi block indices (+j, up to n / b) and the error codes
    (>= 2^30) are disjoint -- a factorisation with >= 1000 blocks reports its
    non-converged block, not a CUDA error."""
    from paper_2002_06960_b200 import randutv as r
    for code in (r.RANDUTV_ERR_CUDA, r.RANDUTV_ERR_ALLOC, r.RANDUTV_ERR_NONFINITE, r.RANDUTV_ERR_CTX,
                 r.RANDUTV_ERR_NCCL, r.RANDUTV_ERR_NOCOMM, r.RANDUTV_ERR_PEER):
        assert code >= 2 ** 30
        assert b"Jacobi" not in lib.randutv_status_string(code)
    for j in (1, 999, 1000, 1005, 65536, 2 ** 30 - 1):
        assert b"Jacobi" in lib.randutv_status_string(j)
    assert lib.randutv_set_option(None, 1, 5) == r.RANDUTV_ERR_CTX
