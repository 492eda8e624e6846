#!/usr/bin/env python
"""Two launches of this library's DGEMM and two of cuBLAS's (torch addmm) on
one c3 shape, for an ncu capture of both kernels side by side:

    ncu --set full -c 4 python tools/gemm_probe.py [rank2b|skinny]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_06960_b200.randutv import Context, colmajor  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "rank2b"
ta, tb, M, N, K, beta = {"rank2b": (0, 1, 16384, 16128, 512, 1.0), "skinny": (1, 0, 16384, 256, 16384, 0.0)}[case]
ctx = Context()
A = colmajor(K, M) if ta else colmajor(M, K)
B = colmajor(N, K) if tb else colmajor(K, N)
C = colmajor(M, N)
for X in (A, B, C):
    X.normal_()
for _ in range(2):
    ctx.randutv_dgemm(ta, tb, A, B, C, alpha=-1.0, beta=beta)
opA = A.t() if ta else A
opB = B.t() if tb else B
for _ in range(2):
    C.addmm_(opA, opB, beta=beta, alpha=-1.0)
torch.cuda.synchronize()
