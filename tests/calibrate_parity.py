"""Rounding-noise calibration of the parity tolerances (run by hand; not collected).

Runs the oracle on A and on A * (1 + 2^-52 N(0,1)) (a backward-error-sized
perturbation) and prints the differences the parity tests measure.  Any
backward-stable implementation -- the GPU path included -- can differ from the
oracle by this much; the tolerances in test_gpu_randutv.py sit >= 30x above it
(DESIGN.md "Parity tolerances").
"""
import numpy as np, sys, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle.randutv import randutv
from paper_2002_06960_b200.inputs import make_numpy
from gpu_util import diag_parity
rng = np.random.default_rng(0)
def pert(A): return np.asfortranarray(A * (1 + 2**-52 * rng.standard_normal(A.shape)))
for (m,n,r,k,b) in [(3000,600,100,160,64),(4096,1024,200,256,64)]:
    A = make_numpy("lowrank", m, n, cfg_index=4, rank=r)
    o1 = randutv(A,b,2,2004,k=k,thin_u=True); o8 = randutv(pert(A),b,2,2004,k=k,thin_u=True)
    print(m,n,r,k, "diag ratio", diag_parity(np.diag(o1["Tk"]), np.diag(o8["Tk"])), "rho rel", abs(o1["rho"]-o8["rho"])/o1["rho"],
          "Tk elem", np.max(np.abs(np.abs(o1["Tk"])-np.abs(o8["Tk"])))/np.linalg.norm(A), "Uk elem", np.max(np.abs(np.abs(o1["Uk"])-np.abs(o8["Uk"]))))
A = make_numpy("powspec", 512, 512, cfg_index=1)
o1 = randutv(A,64,2,2001); o8 = randutv(pert(A),64,2,2001)
print("c1 diag", diag_parity(np.diag(o1["T"]), np.diag(o8["T"])), "T", np.max(np.abs(np.abs(o1["T"])-np.abs(o8["T"]))), "U", np.max(np.abs(np.abs(o1["U"])-np.abs(o8["U"]))), "V", np.max(np.abs(np.abs(o1["V"])-np.abs(o8["V"]))))
for (m,n,b,q) in [(200,200,32,2),(333,333,64,1),(300,170,40,2)]:
    A = np.asfortranarray(np.random.default_rng(m * 1000 + n + b + q).standard_normal((m, n)))
    o1 = randutv(A,b,q,99); o8 = randutv(pert(A),b,q,99)
    print(m,n,b,q,"diag", diag_parity(np.diag(o1["T"]), np.diag(o8["T"])), "T", np.max(np.abs(np.abs(o1["T"])-np.abs(o8["T"])))/np.linalg.norm(A), "U", np.max(np.abs(np.abs(o1["U"])-np.abs(o8["U"]))))
# host-streamed cases (tests/test_gpu_host.py): (520, 520, 64, 2) is the ill-conditioned one
for (m,n,b,q) in [(520,520,64,2),(300,300,32,1),(400,250,40,2)]:
    A = np.asfortranarray(np.random.default_rng(3 * m + n + b).standard_normal((m, n)))
    o1 = randutv(A,b,q,41); o8 = randutv(pert(A),b,q,41)
    print("host", m,n,b,q,"T", np.max(np.abs(np.abs(o1["T"])-np.abs(o8["T"])))/np.linalg.norm(A), "U", np.max(np.abs(np.abs(o1["U"])-np.abs(o8["U"]))), "V", np.max(np.abs(np.abs(o1["V"])-np.abs(o8["V"]))))
