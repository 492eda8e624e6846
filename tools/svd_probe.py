#!/usr/bin/env python
"""One small SVD per width for ncu captures of the Jacobi kernels.  python tools/svd_probe.py W"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_06960_b200.randutv import Context, colmajor  # noqa: E402

w = int(sys.argv[1])
ctx = Context(0)
Bm = colmajor(w, w)
Bm.normal_()
R = torch.linalg.qr(Bm)[1].t().contiguous().t()
for _ in range(3):
    ctx.randutv_small_svd(R)
torch.cuda.synchronize()
print("ok", w)
