"""Kernel variants selected by environment switches, checked against the
default path in subprocesses (the switches are read once per process).

* RUTV_LEAF_PUSH=0: the cluster leaf exchanges its per-column records by a
  cluster barrier + DSMEM loads instead of st.async pushes.  The sums are the
  same values added in the same CTA order, so the panel QR must be BITWISE
  identical.
* RUTV_QR_FUSED=0: the per-leaf S GEMM + t_block + trailing DGEMMs instead of
  the fused panel_update_kernel.  Same mathematics, different summation
  order: agreement within the panel-QR parity bound of test_gpu_kernels.
* RUTV_JACOBI_CLUSTER=0: the L2-staged block Jacobi instead of the cluster
  kernel (register-resident X, W by accumulated 16 x 16 factors): the same
  singular values to the LAPACK bound.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2002_06960_b200.randutv import Context, colmajor
kind, h, w, out = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
ctx = Context(0)
rng = np.random.default_rng(h * 31 + w)
if kind == "qr":
    P0 = rng.standard_normal((h, w))
    P = colmajor(h, w); P.copy_(torch.from_numpy(P0.T.copy()).t())
    _, tau, Tf = ctx.randutv_panel_qr(P)
    np.savez(out, F=P.cpu().numpy(), tau=tau.cpu().numpy(), T=Tf.cpu().numpy())
else:
    B0 = np.triu(rng.standard_normal((w, w)))
    B = colmajor(w, w); B.copy_(torch.from_numpy(B0.T.copy()).t())
    Us, d, Vs, st = ctx.randutv_small_svd(B)
    np.savez(out, d=d.cpu().numpy(), U=Us.cpu().numpy(), V=Vs.cpu().numpy(), B=B0)
"""


def _run(tmp_path, env_extra, kind, h, w, tag):
    out = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, kind, str(h), str(w), out], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("h,w", [(4096, 96), (9000, 64), (12000, 40)])
def test_leaf_push_exchange_is_bitwise_the_barrier_exchange(tmp_path, h, w):
    a = _run(tmp_path, {}, "qr", h, w, "push")
    b = _run(tmp_path, {"RUTV_LEAF_PUSH": "0"}, "qr", h, w, "pull")
    for k in ("F", "tau", "T"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("h,w", [(5000, 128), (777, 45), (16384, 96)])
def test_fused_panel_update_matches_gemm_path(tmp_path, h, w):
    a = _run(tmp_path, {}, "qr", h, w, "fused")
    b = _run(tmp_path, {"RUTV_QR_FUSED": "0"}, "qr", h, w, "gemm")
    tol = 1e-10  # N(0,1) panels: kappa ~ 10, h u kappa with margin (test_gpu_kernels' bound)
    assert np.max(np.abs(a["tau"] - b["tau"])) <= tol
    assert np.max(np.abs(a["F"] - b["F"])) <= tol * max(1.0, np.max(np.abs(b["F"])))
    assert np.max(np.abs(a["T"] - b["T"])) <= tol * max(1.0, np.max(np.abs(b["T"])))
    assert np.all(np.tril(a["T"], -1) == 0.0)


@pytest.mark.parametrize("w", [64, 200, 256])
def test_cluster_jacobi_matches_block_kernel(tmp_path, w):
    a = _run(tmp_path, {}, "svd", 0, w, "cluster")
    b = _run(tmp_path, {"RUTV_JACOBI_CLUSTER": "0"}, "svd", 0, w, "block")
    s = np.linalg.svd(a["B"], compute_uv=False)
    bound = 50 * w * 2.0 ** -53 * s[0]
    assert np.max(np.abs(a["d"] - s)) <= bound
    assert np.max(np.abs(b["d"] - s)) <= bound
    # U_SVD orthogonal to working accuracy on the register-resident path
    U = a["U"]
    assert np.linalg.norm(U.T @ U - np.eye(w), 2) <= 100 * w * 2.0 ** -53
