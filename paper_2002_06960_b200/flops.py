"""Algorithmic flop model of randUTV -- measurement only.

Counts what the method computes per sampled step i (k = i b, r = m - k,
s = n - k), following the steps of Sec. 3.1 / Fig. fig:FLArandutv:
  sample         2 (1 + 2q) r s b
  QR(Y)          3 s b^2 - b^3   (Householder, ~2(sb^2 - b^3/3) + T factor)
  right update   4 m s b + m b^2                       (all m rows)
  V update       4 n s b + n b^2
  QR(col)        3 r b^2 - b^3
  left update    4 r (s-b) b + (s-b) b^2
  U update       4 m r b + m b^2   (forward m x m U)
  folds          2 b^2 (k + s - b) for T, 2 b^2 (m + n) for U, V
final step (s <= b): 3 r s^2 - s^3 + 4 m r s + m s^2 if tall, folds 2 s^2 (k + m + n).
Truncated (K sampled steps) with U_k by backward accumulation replaces the
forward U term by sum_j 4 (m - k_j)(k - k_j) b + 2 b^2 (k - k_j).
The Jacobi SVD (O(b^3) per step) and the RNG are not counted.
Square asymptotics: (12 + 4q)/3 n^3 (T only) + 4 n^3 (U and V).
"""


def sampled_steps(n, b):
    return (n - b + b - 1) // b if n > b else 0


def randutv_flops(m, n, b, q, build_uv=True, k=None):
    b = min(b, n)
    nsamp = sampled_steps(n, b)
    K = nsamp
    with_final = True
    if k is not None:
        K = -(-k // b)
        if K > nsamp:
            K = nsamp
        else:
            with_final = False
    F = 0.0
    for i in range(K):
        kk = i * b
        r, s = m - kk, n - kk
        F += 2 * (1 + 2 * q) * r * s * b
        F += 3 * s * b * b - b ** 3
        F += 4 * m * s * b + m * b * b
        F += 3 * r * b * b - b ** 3
        F += 4 * r * (s - b) * b + (s - b) * b * b
        F += 2 * b * b * (kk + s - b)
        if build_uv:
            F += 4 * n * s * b + n * b * b
            F += 2 * b * b * n
            if k is None:
                F += 4 * m * r * b + m * b * b + 2 * b * b * m
            else:
                F += 4 * r * max(k - kk, 0) * b + 2 * b * b * max(k - kk, 0)
    if with_final:
        kk = K * b
        r, s = m - kk, n - kk
        if s > 0:
            if r > s:
                F += 3 * r * s * s - s ** 3
                if build_uv:
                    F += 4 * m * r * s + m * s * s
            F += 2 * s * s * kk
            if build_uv:
                F += 2 * s * s * (m + n)
    return float(F)


def hqrrp_flops(m, n, b, build_q=True):
    """Algorithmic flop model of HQRRP (Sec. 2) per step (k = i b,
    r = m - k, s = n - k, w = min(b, s)): sketch 2 b r s, sketch CPQR
    ~ 2 b^2 s, panel QR 2 r w^2 - 2 w^3 / 3, left update 4 r (s - w) w, and the
    Q update 4 m r w when Q is built."""
    b = min(b, n)
    F = 0.0
    for k in range(0, n, b):
        r, s = m - k, n - k
        w = min(b, s)
        F += 2.0 * b * r * s + 2.0 * b * b * s + 2.0 * r * w * w - 2.0 * w ** 3 / 3 + 4.0 * r * (s - w) * w
        if build_q:
            F += 4.0 * m * r * w
    return F


def host_stream_traffic(m, n, b, q, cache_panels, policy="lru"):
    """PCIe bytes of the host-streamed T-only randUTV (csrc/host.cu, S12) --
    measurement only: replays the panel access sequence of the driver (per
    sampled step i, k = i b: [step 0 only: the S2 pass over rows k:m], 2q power
    passes over rows k:m, the T W_V read pass over all rows, panel i read +
    written, one read-write pass over panels > i; pass directions alternate,
    starting forward on even steps; final block read + written) through a
    cache of `cache_panels` slots and returns (h2d_bytes, d2h_bytes).

    policy "lru" is the driver's (least recently used, one-panel prefetch
    modelled as an access); "belady" evicts the resident panel whose next use
    lies farthest ahead (the optimal offline policy, the access sequence being
    known in advance -- SURVEY.md §8(d) M7).  Also "none": no cache (every
    access loads, every write-back stores) -- M7's algorithmic floor."""
    b = min(b, n)
    np_ = -(-n // b)
    width = [min(b, n - j * b) for j in range(np_)]
    seq = []   # (panel, lo, dirty)
    nsamp = sampled_steps(n, b)
    for i in range(nsamp):
        k = i * b
        fwd = (i % 2 == 0)

        def pass_(p0, lo, dirty):
            nonlocal fwd
            order = range(p0, np_) if fwd else range(np_ - 1, p0 - 1, -1)
            fwd = not fwd
            for j in order:
                seq.append((j, lo, dirty))
        if i == 0:
            pass_(i, k, False)
        for _ in range(2 * q):
            pass_(i, k, False)
        pass_(i, 0, False)
        seq.append((i, 0, True))
        pass_(i + 1, 0, True)
    seq.append((nsamp, 0, True))
    if policy == "none":
        h2d = sum((m - lo) * width[j] * 8 for j, lo, _ in seq)
        d2h = sum(m * width[j] * 8 for j, _, d in seq if d)
        return float(h2d), float(d2h)
    # next-use index per position (Belady)
    nxt = [0] * len(seq)
    last = {}
    for t in range(len(seq) - 1, -1, -1):
        j = seq[t][0]
        nxt[t] = last.get(j, 1 << 62)
        last[j] = t
    res = {}   # panel -> [lo, dirty, last_use, next_use]
    h2d = d2h = 0
    for t, (j, lo, dirty) in enumerate(seq):
        if j in res:
            e = res[j]
            if lo < e[0]:
                h2d += (e[0] - lo) * width[j] * 8
                e[0] = lo
        else:
            if len(res) >= cache_panels:
                if policy == "belady":
                    v = max(res, key=lambda p: res[p][3])
                else:
                    v = min(res, key=lambda p: res[p][2])
                ev = res.pop(v)
                if ev[1]:
                    d2h += (m - ev[0]) * width[v] * 8
            h2d += (m - lo) * width[j] * 8
            res[j] = [lo, False, t, 0]
        e = res[j]
        e[1] = e[1] or dirty
        e[2] = t
        e[3] = nxt[t]
    for j, e in res.items():
        if e[1]:
            d2h += (m - e[0]) * width[j] * 8
    return float(h2d), float(d2h)
