#!/usr/bin/env python
"""Per-kernel timing of the library's step entries through the C ABI (CUDA
events recorded by the library on the ctx stream).  Development tool for the
roofline work: prints one JSON line per case.

    python tools/bench_kernels.py [gemm] [qr] [svd]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2002_06960_b200.randutv import Context, colmajor  # noqa: E402


def timed(ctx, fn, kind, reps=5):
    fn()
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    p = ctx.profile()[kind]
    ctx.set_profiling(False)
    return p


def gemm_cases(ctx):
    # (label, ta, tb, M, N, K): the c3 iteration-0 shapes and their c2 analogues
    cases = [("S2 Y=At^T G c3", 1, 0, 16384, 256, 16384), ("S3 Z=At Y c3", 0, 0, 16384, 256, 16384),
             ("S5 Z=X W c3", 0, 0, 16384, 256, 16384), ("S5 X-=Z2 W^T c3", 0, 1, 16384, 16384, 256),
             ("S7 Z=W^T X c3", 1, 0, 256, 16128, 16384), ("S7 X-=W Z2 c3", 0, 0, 16384, 16128, 256),
             ("S5 X-=Z2 W^T c2", 0, 1, 4096, 4096, 128), ("square 8192", 0, 0, 8192, 8192, 8192)]
    for label, ta, tb, M, N, K in cases:
        A = colmajor(K, M) if ta else colmajor(M, K)
        B = colmajor(N, K) if tb else colmajor(K, N)
        C = colmajor(M, N)
        A.normal_()
        B.normal_()
        C.normal_()
        p = timed(ctx, lambda: ctx.randutv_dgemm(ta, tb, A, B, C, alpha=-1.0, beta=1.0), "dgemm")
        ms = p["ms"] / 5
        print(json.dumps({"kernel": "dgemm", "case": label, "M": M, "N": N, "K": K, "ms": round(ms, 4),
                          "tflops": round(2 * M * N * K / (ms * 1e-3) / 1e12, 3), "launches": p["launches"] / 5}))
        del A, B, C


def cublas_cases():
    """torch.matmul (cuBLAS DGEMM) on the same shapes: the library-GEMM reference point."""
    cases = [("S2 Y=At^T G c3", 1, 0, 16384, 256, 16384), ("S5 X-=Z2 W^T c3", 0, 1, 16384, 16384, 256),
             ("S7 X-=W Z2 c3", 0, 0, 16384, 16128, 256), ("square 8192", 0, 0, 8192, 8192, 8192)]
    for label, ta, tb, M, N, K in cases:
        A = colmajor(K, M) if ta else colmajor(M, K)
        B = colmajor(N, K) if tb else colmajor(K, N)
        C = colmajor(M, N)
        A.normal_()
        B.normal_()
        C.normal_()
        opA = A.t() if ta else A
        opB = B.t() if tb else B
        f = lambda: C.addmm_(opA, opB, beta=1.0, alpha=-1.0)
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"kernel": "cublas_dgemm", "case": label, "M": M, "N": N, "K": K, "ms": round(ms, 4),
                          "tflops": round(2 * M * N * K / (ms * 1e-3) / 1e12, 3)}))
        del A, B, C


def gemm_diag(ctx):
    """Separates main-loop from per-tile (prologue + epilogue) cost of the rank-b update."""
    M = N = 16384
    for K in (64, 128, 256, 512, 1024, 2048):
        for beta in (0.0, 1.0):
            A = colmajor(M, K)
            B = colmajor(N, K)
            C = colmajor(M, N)
            A.normal_()
            B.normal_()
            C.normal_()
            p = timed(ctx, lambda: ctx.randutv_dgemm(0, 1, A, B, C, alpha=-1.0, beta=beta), "dgemm")
            ms = p["ms"] / 5
            print(json.dumps({"kernel": "dgemm_diag", "M": M, "N": N, "K": K, "beta": beta, "ms": round(ms, 4),
                              "tflops": round(2 * M * N * K / (ms * 1e-3) / 1e12, 3)}))
            del A, B, C


def qr_cases(ctx):
    for h, w in [(16384, 256), (12288, 256), (8192, 256), (20000, 256), (65536, 512), (4096, 128)]:
        P0 = colmajor(h, w)
        P0.normal_()
        P = colmajor(h, w)

        def run():
            P.copy_(P0)
            ctx.randutv_panel_qr(P)
        ctx.set_profiling(True)
        run()
        torch.cuda.synchronize()
        ctx.set_profiling(False)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        total = e0.elapsed_time(e1) / 3
        ctx.set_profiling(True)
        run()
        torch.cuda.synchronize()
        prof = ctx.profile()
        ctx.set_profiling(False)
        print(json.dumps({"kernel": "panel_qr", "h": h, "w": w, "total_ms": round(total, 3),
                          "leaf_ms": round(prof["qr_leaf"]["ms"], 3), "leaf_launches": prof["qr_leaf"]["launches"],
                          "gemm_ms": round(prof["dgemm"]["ms"], 3), "gemm_launches": prof["dgemm"]["launches"],
                          "leaf_GBps": round(prof["qr_leaf"]["bytes"] / (prof["qr_leaf"]["ms"] * 1e-3) / 1e9, 1)}))


def svd_cases(ctx):
    for w in (64, 128, 256, 512):
        Bm = colmajor(w, w)
        Bm.normal_()
        Q, R = torch.linalg.qr(Bm)
        R = R.t().contiguous().t()
        p = timed(ctx, lambda: ctx.randutv_small_svd(R), "jacobi", reps=3)
        print(json.dumps({"kernel": "jacobi_svd", "w": w, "ms": round(p["ms"] / 3, 3)}))


if __name__ == "__main__":
    torch.cuda.set_device(0)
    ctx = Context(0)
    which = sys.argv[1:] or ["gemm", "qr", "svd"]
    if "gemm" in which:
        gemm_cases(ctx)
    if "cublas" in which:
        cublas_cases()
    if "gemmdiag" in which:
        gemm_diag(ctx)
    if "qr" in which:
        qr_cases(ctx)
    if "svd" in which:
        svd_cases(ctx)
