#!/usr/bin/env python
"""The largest out-of-core run the GPU box can hold:
n = 131072 (137 GB, T only, q = 1, b = 512) from ONE pinned host copy through
a bounded device panel cache, next to the same factorisation resident in HBM
(T overwrites A).  Guards the host memory before pinning.  One JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_06960_b200.flops import host_stream_traffic, randutv_flops  # noqa: E402
from paper_2002_06960_b200.randutv import RANDUTV_NO_UV, Context, colmajor, pinned_colmajor  # noqa: E402

n = int(os.environ.get("OOC_N", "131072"))
b, q, seed = 512, 1, 2005
cache_gib = float(os.environ.get("OOC_CACHE_GIB", "48"))
need = 8 * n * n
avail = 0
for l in open("/proc/meminfo"):
    if l.startswith("MemAvailable:"):
        avail = int(l.split()[1]) * 1024
if avail < need * 1.15:
    print(json.dumps({"skipped": f"host MemAvailable {avail / 1e9:.0f} GB < 1.15 x {need / 1e9:.0f} GB"}))
    sys.exit(0)
ctx = Context(0)
F = randutv_flops(n, n, b, q, build_uv=False)


def make():
    g = torch.Generator(device="cuda")
    g.manual_seed(1005)
    A = colmajor(n, n)
    A.normal_(generator=g)
    return A


# compute-only reference: the same T-only factorisation in HBM, T overwriting A
A = make()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.randutv_factor_ex(A, b, q, seed, build_uv=False, T=A)
e1.record()
torch.cuda.synchronize()
comp_s = e0.elapsed_time(e1) * 1e-3
diag_hbm = torch.diagonal(A)[:1024].abs().cpu().numpy()
del A
torch.cuda.empty_cache()
# the host copy
A = make()
t0 = time.time()
Ah = pinned_colmajor(n, n)
pin_s = time.time() - t0
torch.from_numpy(Ah.T).copy_(A.t())
del A
torch.cuda.empty_cache()
_, _, rep = ctx.randutv_factor_host(Ah, b, q, seed, build_uv=False, cache_bytes=int(cache_gib * 2 ** 30))
real_s = rep["wall_ms"] * 1e-3
diag_host = np.abs(np.diag(Ah[:1024, :1024]))
hm, dm = host_stream_traffic(n, n, b, q, rep["cache_slots"], "belady")
print(json.dumps({
    "workload": f"n={n} Gaussian (A {need / 1e9:.0f} GB), b={b}, q={q}, T only, one pinned host copy",
    "device_cache_gib": cache_gib, "cache_slots": rep["cache_slots"], "host_pin_s": round(pin_s, 1),
    "computational_time_s": round(comp_s, 2), "real_time_s": round(real_s, 2),
    "real_over_comp": round(real_s / comp_s, 3),
    "tflops_host": round(F / real_s / 1e12, 2), "tflops_hbm": round(F / comp_s / 1e12, 2),
    "h2d_bytes": rep["h2d_bytes"], "d2h_bytes": rep["d2h_bytes"], "model_belady_h2d": hm, "model_belady_d2h": dm,
    "h2d_GBps": rep["h2d_bytes"] / (rep["h2d_ms"] * 1e-3) / 1e9 if rep["h2d_ms"] else None,
    "diag_first_1024_max_rel_diff_host_vs_hbm": float(np.max(np.abs(diag_host - diag_hbm) / diag_hbm)),
}))
