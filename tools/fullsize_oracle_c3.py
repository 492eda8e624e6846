#!/usr/bin/env python
"""One-off full-size parity of the c3 workload (n = 16384, b = 256, q = 2, U and V):
the GPU's complete factorisation against the oracle's complete factorisation of
the same A bytes (all 64 steps; ~30 min of the box's host cores), at the
north-star bounds, plus the rounding-noise band of the
GPU itself (A vs A(1 + 2^-52 E)) for the elementwise comparisons.  Writes
one JSON record (profiles/parity_c3_full_r02.json)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gpu_util import diag_parity  # noqa: E402
from oracle.randutv import randutv as oracle_randutv  # noqa: E402
from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch  # noqa: E402
from paper_2002_06960_b200.randutv import Context  # noqa: E402

c = CONFIGS["c3"]
m, n, b, q, seed = c["m"], c["n"], c["b"], c["q"], 2003
ctx = Context()
A = make_config_torch("c3")
nA = float(torch.linalg.norm(A))
U, T, V, st = ctx.randutv_factor_ex(A, b, q, seed)
g = torch.Generator(device=A.device)
g.manual_seed(7)
E = torch.randn(n, m, generator=g, device=A.device, dtype=torch.float64).t()
Up, Tp, Vp, _ = ctx.randutv_factor_ex(A * (1 + 2.0 ** -52 * E), b, q, seed)
del E
torch.cuda.synchronize()
tonp = lambda X: X.cpu().numpy()
Tg, Ug, Vg = tonp(T), tonp(U), tonp(V)
Tpn, Upn, Vpn = tonp(Tp), tonp(Up), tonp(Vp)
del U, T, V, Up, Tp, Vp
Ah = A.cpu().numpy()
del A
torch.cuda.empty_cache()
t0 = time.time()
o = oracle_randutv(np.array(Ah, order="F"), b, q, seed)
t_or = time.time() - t0
e = lambda X, Y: float(np.max(np.abs(np.abs(X) - np.abs(Y))))
dg, dp, do = np.abs(np.diag(Tg)), np.abs(np.diag(Tpn)), np.abs(np.diag(o["T"]))
rec = {
    "config": "c3 full: n=16384, b=256, q=2, U and V, all 64 steps",
    "oracle_seconds": round(t_or, 1),
    "diag_A16_max_ratio": diag_parity(dg, do),
    "diag_A16_band_gpu": diag_parity(dg, dp),
    "diag_rel_max": float(np.max(np.abs(dg - do) / do)),
    "T_elem_over_normA": e(Tg, o["T"]) / nA, "T_band": e(Tg, Tpn) / nA,
    "U_elem": e(Ug, o["U"]), "U_band": e(Ug, Upn),
    "V_elem": e(Vg, o["V"]), "V_band": e(Vg, Vpn),
    "sum_log10_diag_gpu": float(np.sum(np.log10(dg))), "sum_log10_diag_oracle": float(np.sum(np.log10(do))),
    "tril_zero": bool(np.all(np.tril(Tg, -1) == 0.0)),
}
# reconstruction and orthogonality on the GPU side (torch, test-side only)
Ad, Ud, Td, Vd = (torch.from_numpy(np.ascontiguousarray(X)).cuda() for X in (Ah, Ug, Tg, Vg))
rec["recon"] = float(torch.linalg.norm(Ad - (Ud @ Td) @ Vd.t()) / torch.linalg.norm(Ad))
for name, Q in (("orthU", Ud), ("orthV", Vd)):
    Eq = Q.t() @ Q
    Eq.diagonal().sub_(1.0)
    rec[name] = float(torch.linalg.eigvalsh(Eq).abs().max())
print(json.dumps(rec))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rec, open("gpurun_out/parity_c3_full_r02.json", "w"), indent=1)
