#!/usr/bin/env python
"""Measured PCIe bytes of the host-streamed T-only randUTV against the replay
model paper_2002_06960_b200.flops.host_stream_traffic (Belady / LRU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_06960_b200.flops import host_stream_traffic  # noqa: E402
from paper_2002_06960_b200.randutv import Context, pinned_colmajor  # noqa: E402

policy = "lru" if os.environ.get("RUTV_HOST_EVICT") == "lru" else "belady"
ctx = Context(0)
for (m, n, b, q, C) in [(2048, 2048, 128, 1, 5), (3000, 2500, 128, 2, 8), (4096, 4096, 256, 1, 7), (4096, 4096, 128, 1, 12)]:
    A = pinned_colmajor(m, n)
    A[:] = np.random.default_rng(m + n).standard_normal((m, n))
    slot = max(m, n) * b * 8
    slot = ((max(m, n) * b + 31) // 32) * 32 * 8
    _, _, rep = ctx.randutv_factor_host(A, b, q, 3, build_uv=False, cache_bytes=C * slot)
    h, d = host_stream_traffic(m, n, b, q, rep["cache_slots"], policy)
    print(json.dumps({"m": m, "n": n, "b": b, "q": q, "slots": rep["cache_slots"], "policy": policy,
                      "h2d": rep["h2d_bytes"], "h2d_model": h, "d2h": rep["d2h_bytes"], "d2h_model": d}))
