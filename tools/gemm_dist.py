#!/usr/bin/env python
"""Summarise a RUTV_PROF_DUMP per-launch log: time and efficiency by GEMM shape class.

    RUTV_PROF_DUMP=/tmp/p.txt python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
    python tools/gemm_dist.py /tmp/p.txt
"""
import collections
import sys

rows = [l.split() for l in open(sys.argv[1])]
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
kinds = {0: "dgemm", 1: "qr_leaf", 2: "jacobi", 3: "gaussian"}
for r in rows:
    kind, m, n, k, ms, fl = int(r[0]), int(r[1]), int(r[2]), int(r[3]), float(r[4]), float(r[5])
    if kind != 0:
        key = kinds.get(kind, str(kind))
    else:
        small = min(m, n)
        if k <= 64:
            key = f"gemm K<=64"
        elif small <= 64:
            key = "gemm tiny side<=64 (QR internals)"
        elif k <= 512 and small > 512:
            key = f"gemm rank-{'b' if k <= 256 else '2b'} update (K={'<=256' if k <= 256 else '<=512'})"
        elif small <= 512:
            big = max(m, n)
            key = "gemm skinny (one side <= 512, long K)" + (" big>=8192" if big >= 8192 and k >= 8192 else " smaller")
        else:
            key = "gemm other"
    t = tot[key]
    t[0] += 1
    t[1] += ms
    t[2] += fl
T = sum(v[1] for v in tot.values())
print(f"{'class':42s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'TF/s':>7s}")
for key, (c, ms, fl) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{key:42s} {c:8d} {ms:9.1f} {ms / T:6.1%} {fl / (ms * 1e-3) / 1e12 if ms else 0:7.2f}")

# the heaviest individual shapes (M, N, K) by summed time, with their rate
if len(sys.argv) > 2:
    shp = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows:
        if int(r[0]) != 0:
            continue
        key = (int(r[1]), int(r[2]), int(r[3]))
        shp[key][0] += 1
        shp[key][1] += float(r[4])
        shp[key][2] += float(r[5])
    print(f"\n{'M':>7s} {'N':>7s} {'K':>7s} {'launches':>8s} {'ms':>8s} {'TF/s':>7s}")
    for (m, n, k), (c, ms, fl) in sorted(shp.items(), key=lambda x: -x[1][1])[:int(sys.argv[2])]:
        print(f"{m:7d} {n:7d} {k:7d} {c:8d} {ms:8.2f} {fl / (ms * 1e-3) / 1e12 if ms else 0:7.2f}")
