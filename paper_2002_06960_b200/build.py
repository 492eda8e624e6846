"""Build librandutv.so in-tree with nvcc for sm_100a (no torch in the ABI)."""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# RUTV_BUILD_OUT / RUTV_NVCC_EXTRA: build a variant library elsewhere (A/B tuning only)
OUT = os.environ.get("RUTV_BUILD_OUT", os.path.join(HERE, "librandutv.so"))
EXTRA = os.environ.get("RUTV_NVCC_EXTRA", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]
SOURCES = ["philox.cu", "dgemm.cu", "qr.cu", "jacobi.cu", "misc.cu", "randutv.cu", "dist.cu", "host.cu", "hqrrp.cu"]


def nccl_dir():
    """The NCCL headers/library torch ships (nvidia-nccl wheel): headers at build
    time, libnccl.so.2 loaded at run time by dist.cu (dlopen, no link dependency)."""
    for p in sys.path:
        d = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (nvidia/nccl/include in site-packages)")


def _compile(src, objdir, verbose):
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    extra = []
    if src == "dist.cu":
        d = nccl_dir()
        extra = ["-I", os.path.join(d, "include"),
                 f'-DRUTV_NCCL_PATH="{os.path.join(d, "lib", "libnccl.so.2")}"']
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False, force=False):
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "driver.cuh"), os.path.join(HERE, "..", "include", "randutv.h")]
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(p) < t for p in srcs + hdrs + [__file__]):
            return OUT
    objdir = os.path.join(HERE, "build") if OUT == os.path.join(HERE, "librandutv.so") else OUT + ".objs"
    os.makedirs(objdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, objdir, verbose), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    tmp = OUT + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
