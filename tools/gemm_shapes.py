#!/usr/bin/env python
"""DGEMM shape sweep over a c3 factorisation (n = 16384, b = 256): the step-i
shapes of every GEMM class (skinny sample / T W / W^T X products, rank-b and
rank-2b updates), this library's kernel (through randutv_dgemm, split-K
workspace included) against cuBLAS (torch addmm) on the same operands.
One JSON line per (step, class).  Development tool for the DGEMM roofline."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_06960_b200.randutv import Context, colmajor  # noqa: E402

n, b = 16384, 256
steps = [int(x) for x in os.environ.get("STEPS", "0,8,16,24,32,40,48,56,60").split(",")]
ctx = Context()


def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for i in steps:
    r = s = n - b * i
    cases = [("S2 TN A^T G", 1, 0, s, b, r, 0.0), ("S3 NN A Y", 0, 0, r, b, s, 0.0),
             ("S5 NN X W", 0, 0, n, b, s, 0.0), ("S7 TN X^T W", 1, 0, s - b, b, r, 0.0),
             ("rank-b NT", 0, 1, n, s, b, 1.0), ("rank-2b NT", 0, 1, r, s - b, 2 * b, 1.0),
             ("m x b x b NN (Z T_V)", 0, 0, r, b, b, 0.0)]
    for label, ta, tb, M, N, K, beta in cases:
        if M <= 0 or N <= 0 or K <= 0:
            continue
        A = colmajor(K, M) if ta else colmajor(M, K)
        B = colmajor(N, K) if tb else colmajor(K, N)
        C = colmajor(M, N)
        A.normal_()
        B.normal_()
        C.normal_()
        # ours: the library's own per-launch events (randutv_dgemm synchronises
        # after every call, so wall-clock events would include that)
        f = lambda: ctx.randutv_dgemm(ta, tb, A, B, C, alpha=-1.0, beta=beta)
        f()
        ctx.set_profiling(True)
        for _ in range(5):
            f()
        ours = ctx.profile()["dgemm"]["ms"] / 5
        ctx.set_profiling(False)
        opA = A.t() if ta else A
        opB = B.t() if tb else B
        cub = timeit(lambda: C.addmm_(opA, opB, beta=beta, alpha=-1.0))
        fl = 2.0 * M * N * K
        print(json.dumps({"step": i, "case": label, "M": M, "N": N, "K": K, "ours_ms": round(ours, 4),
                          "ours_TF": round(fl / ours / 1e9, 2), "cublas_TF": round(fl / cub / 1e9, 2)}), flush=True)
        del A, B, C
