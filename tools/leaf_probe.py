#!/usr/bin/env python
"""One panel QR per height (a single 32-column leaf) for ncu captures of the
QR leaf kernel variants.  python tools/leaf_probe.py H [W]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_06960_b200.randutv import Context, colmajor  # noqa: E402

h = int(sys.argv[1])
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = Context(0)
P0 = colmajor(h, w)
P0.normal_()
P = colmajor(h, w)
for _ in range(3):
    P.copy_(P0)
    ctx.randutv_panel_qr(P)
torch.cuda.synchronize()
print("ok", h, w)
