import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, time, json
from paper_2002_06960_b200.randutv import Context, colmajor
c = Context()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for (r, s, b) in [(16384, 16384, 256), (8192, 8192, 256), (4096, 4096, 256)]:
    A = colmajor(r, s); A.normal_(); G = colmajor(r, b); G.normal_()
    Y1 = colmajor(b, s); Y2 = colmajor(s, b)
    ms1 = t(lambda: c.randutv_dgemm(True, False, G, A, Y1))   # Y = G^T A  (M = b small)
    ms2 = t(lambda: c.randutv_dgemm(True, False, A, G, Y2))   # Y^T = A^T G (N = b small)
    fl = 2.0 * r * s * b
    print(json.dumps({"r": r, "s": s, "b": b, "GtA_ms": round(ms1, 3), "GtA_TF": round(fl / ms1 / 1e9, 1),
                      "AtG_ms": round(ms2, 3), "AtG_TF": round(fl / ms2 / 1e9, 1)}))
