#!/usr/bin/env python
"""Benchmark of the B200 randUTV hot path (BASELINE.json metric: randUTV FP64
GFLOP/s and t/n^3 at 1/2/4/8 B200; % of FP64 tensor peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A "step" is one full randUTV factorisation (every row of SURVEY.md §8(a):
S1-S10, U and V built) of the config's seeded synthetic matrix, resident in HBM.
Default workload: c3 (n = 16384, b = 256, q = 2, exponential spectrum), the
largest config quoted at 1/2/4/8 GPUs that a single step of finishes in
seconds (DESIGN.md §Measurement explains the choice; c2 and c5 run with
--config).  value = F_model / t (GFLOP/s, F from paper_2002_06960_b200.flops),
whole job over all ranks.  Multi-GPU (N > 1, torchrun): ONE factorisation of
the same matrix sharded over the N GPUs (1-D block-cyclic column blocks, NCCL
AllReduce / AllGather / Broadcast) -- "scaling": "strong".

--impl reference times the CPU oracle (oracle/, numpy) on the host cores on a
bounded sample of the same workload (the first sampled step of the config) --
the only other place this script executes oracle/ besides the cpu_baseline leg.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
NCU_TRAFFIC_FILE = os.path.join(ROOT, "profiles", "dgemm_traffic.json")
METRIC = "randUTV FP64 GFLOP/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-profile", action="store_true", help="do not record per-kernel CUDA events")
    p.add_argument("--mode", default="hbm", choices=["hbm", "host"],
                   help="host: the host-streamed (out-of-core analogue) entry, A/U/V in pinned host memory")
    p.add_argument("--cache-gib", type=float, default=None,
                   help="device panel cache for --mode host (default: a quarter of A)")
    p.add_argument("--no-uv", action="store_true", help="T only (the paper's 'no orthonormal matrices')")
    p.add_argument("--q", type=int, default=None,
                   help="--mode host only: override the config's power steps (the paper's Table 1 runs use q = 0)")
    p.add_argument("--no-graph", dest="graph", action="store_false",
                   help="time eager calls instead of replays of one captured RANDUTV_ASYNC factorisation "
                        "(CUDA graph; the default for full single-GPU factorisations)")
    p.add_argument("--reorth", action="store_true",
                   help="RANDUTV_REORTH: re-orthonormalised power steps (NEXT-4; extra QRs not in the flop model)")
    p.add_argument("--algo", default="randutv", choices=["randutv", "hqrrp"],
                   help="hqrrp: the paper's column-pivoted QR (Sec. 2, SURVEY §8(f) NEXT-3) on the config's matrix")
    p.add_argument("--sharded", action="store_true",
                   help="use the column-sharded NCCL path even on one GPU (exercises the N > 1 code path)")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        import statistics
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ----------------------------------------------------------------------------- helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def fp64_peak():
    """Measured FP64 DMMA sustained peak (tools/fp64_peak.cu on this pool's B200)."""
    try:
        d = json.load(open(FP64_PEAK_FILE))
        return float(d["dmma884_sustained_tflops"]), "measured (profiles/fp64_peak_r01.json, DMMA sustained)"
    except Exception:
        return 37.2, "nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz (measurement file missing)"


SAMPLE_FLOPS = 6e11  # ~20 s of the numpy oracle on a 16-32 core host


def sample_shape(cfg_name):
    """Leading m_s x n_s block of the config (its aspect ratio, b and q) whose first
    sampled step costs about SAMPLE_FLOPS under the flop model."""
    from paper_2002_06960_b200.flops import randutv_flops
    from paper_2002_06960_b200.inputs import CONFIGS
    c = CONFIGS[cfg_name]
    m, n, b, q = c["m"], c["n"], c["b"], c["q"]
    f = 1.0
    while True:
        ms, ns = max(int(m * f) // b * b, 2 * b), max(int(n * f) // b * b, 2 * b)
        if randutv_flops(ms, ns, b, q, build_uv=True, k=b) <= SAMPLE_FLOPS or ns <= 2 * b:
            return ms, ns
        f *= 0.9


def cpu_sample(cfg_name, A_host, seed):
    """The oracle (as it stands) on a bounded sample of the workload: the first
    sampled step (truncated k = b, thin U) of the config's leading m_s x n_s block,
    timed on this host's cores."""
    from threadpoolctl import threadpool_info

    from oracle.randutv import randutv as oracle_randutv
    from paper_2002_06960_b200.flops import randutv_flops
    from paper_2002_06960_b200.inputs import CONFIGS
    c = CONFIGS[cfg_name]
    b, q = c["b"], c["q"]
    import numpy as np
    ms, ns = sample_shape(cfg_name)
    As = np.asfortranarray(A_host[:ms, :ns])
    t0 = time.perf_counter()
    oracle_randutv(As, b, q, seed, k=b, thin_u=True)
    dt = time.perf_counter() - t0
    F = randutv_flops(ms, ns, b, q, build_uv=True, k=b)
    threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    # the whole configuration at the sample's rate (labelled: an extrapolation,
    # the oracle is never run on the full matrix here)
    k = c.get("k") if not c.get("full", True) else None
    F_full = randutv_flops(c["m"], c["n"], b, q, build_uv=True, k=k)
    return {"value": F / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
            "rate_of": "the bounded sample below (GFLOP/s of the flop model on the sample), not of the full config",
            "sample": f"{cfg_name}: first sampled step (truncated k=b={b}, q={q}, V + thin U_k) of the leading "
                      f"{ms}x{ns} block, {F:.3g} flops in {dt:.1f} s (numpy/OpenBLAS, {threads} threads, "
                      f"{os.cpu_count()} host cpus)",
            "extrapolated_full_config_s": round(F_full / (F / dt), 1),
            "seconds": dt, "flops": F}


def config_dict(name, ws, sharded=None):
    """The workload description shared by both arms."""
    from paper_2002_06960_b200.flops import randutv_flops
    from paper_2002_06960_b200.inputs import CONFIGS
    c = CONFIGS[name]
    m, n, b, q = c["m"], c["n"], c["b"], c["q"]
    k = c.get("k") if not c.get("full", True) else None
    sharded = ws > 1 if sharded is None else sharded
    return {"workload": f"{name}: " + {
        "c1": "n=512 known spectrum", "c2": "n=4096 Gaussian", "c3": "n=16384 exp spectrum",
        "c4": "262144x8192 low-rank + noise", "c5": "n=65536 Gaussian"}[name]
        + f", b={b}, q={q}, " + (f"truncated rank-{k} randUTV (U_k, T_k, V)" if k else "full randUTV with U and V"),
        "m": m, "n": n, "b": b, "q": q, "flops_per_step": randutv_flops(m, n, b, q, build_uv=True, k=k),
        "parallelism": f"column-sharded x{ws} (1-D block-cyclic, NCCL)" if sharded else "single",
        "l2": "inputs larger than L2 (A is %.2f GB, L2 126 MB); no flush" % (8 * m * n / 1e9)
        if 8 * m * n > 126e6 else "input fits L2: not flushed"}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    from paper_2002_06960_b200.inputs import CONFIGS, make_numpy
    cfg = CONFIGS[args.config]
    # the config's recipe (kind, seeds) at the bounded sample size: a leading
    # block of the full matrix would need its n x n Haar factors on the host
    ms, ns = sample_shape(args.config)
    A = make_numpy(cfg["kind"], ms, ns, cfg_index=int(args.config[1:]))
    seed = 2000 + int(args.config[1:])
    times = []
    cs = None
    for _ in range(max(args.warmup, 0)):
        cs = cpu_sample(args.config, A, seed)
    for _ in range(args.steps):
        cs = cpu_sample(args.config, A, seed)
        times.append(cs["seconds"])
    t = sum(times) / len(times)
    val = cs["flops"] / t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, ws),
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cs["cores"], "kind": "oracle",
                             "sample": cs["sample"], "rate_of": cs["rate_of"],
                             "extrapolated_full_config_s": cs["extrapolated_full_config_s"]},
            "ms_per_step_is": "the oracle's time for the bounded sample (cpu_baseline.sample)",
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch

    from paper_2002_06960_b200.flops import randutv_flops
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    from paper_2002_06960_b200.randutv import Context, colmajor, randutv_factor

    ws, rank, local = dist_env()
    sharded = ws > 1 or args.sharded
    if sharded:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if ws == 1 and "MASTER_ADDR" not in os.environ:
            os.environ["MASTER_ADDR"] = "127.0.0.1"
            os.environ["MASTER_PORT"] = os.environ.get("MASTER_PORT", "29531")
            os.environ["RANK"], os.environ["WORLD_SIZE"] = "0", "1"
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cfg = CONFIGS[args.config]
    m, n, b, q = cfg["m"], cfg["n"], cfg["b"], cfg["q"]
    seed = 2000 + int(args.config[1:])
    trunc_k = cfg.get("k") if not cfg.get("full", True) else None
    F = randutv_flops(m, n, b, q, build_uv=True, k=trunc_k)

    A = make_config_torch(args.config, device=f"cuda:{dev}")
    stream = torch.cuda.Stream()
    ctx = Context(dev, stream)
    if sharded:
        # column-sharded path: block-cyclic columns of A, row
        # ranges of U and V; NCCL communicator bootstrapped over torch.distributed
        from paper_2002_06960_b200.randutv import dist_layout, local_columns
        ctx.comm_init_torch()
        lay = dist_layout(m, n, b, ws, rank)
        cols = torch.from_numpy(local_columns(n, b, ws, rank)).to(A.device)
        A_loc = colmajor(m, lay["ncols"])
        A_loc.copy_(A.index_select(1, cols))
        del A
        torch.cuda.empty_cache()
        T_loc = colmajor(m, lay["ncols"])
        U_loc = colmajor(lay["u1"] - lay["u0"], trunc_k if trunc_k else m)
        V_loc = colmajor(lay["v1"] - lay["v0"], n)

        def step():
            T_loc.copy_(A_loc)
            if trunc_k:
                ctx.randutv_factor_dist_rank(T_loc, m, n, trunc_k, b, q, seed, Uk_local=U_loc, V_local=V_loc)
            else:
                ctx.randutv_factor_dist(T_loc, m, n, b, q, seed, U_local=U_loc, V_local=V_loc)
    elif trunc_k is not None:
        def step():
            ctx.randutv_factor_rank(A, trunc_k, b, q, seed)
    else:
        T = colmajor(m, n)
        U = colmajor(m, m)
        V = colmajor(n, n)

        fl = 4 if args.reorth else 0  # RANDUTV_REORTH

        def step():
            ctx.randutv_factor_ex(A, b, q, seed, U=U, T=T, V=V, flags=fl)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    graph_launches = None
    if args.graph and trunc_k is not None:
        args.graph = False  # graphs are captured for the full factorisation only

    def async_call():
        # the step as one RANDUTV_ASYNC call (no host synchronisation inside):
        # single-GPU, or the sharded NCCL path (its collectives are captured too)
        if sharded:
            T_loc.copy_(A_loc)
            ctx.randutv_factor_dist(T_loc, m, n, b, q, seed, U_local=U_loc, V_local=V_loc, flags=8)
        else:
            ctx.randutv_factor_ex(A, b, q, seed, U=U, T=T, V=V, flags=fl | 8)  # RANDUTV_ASYNC
    if args.graph:
        # the whole factorisation (main, side and V streams) as one CUDA graph.
        # Two captures of the same call: g without and gp with the per-launch
        # profiling events (external event-record nodes, re-recorded by every
        # replay).  The timed region replays g for steps 1..K-1 and gp for the
        # last step, whose events randutv_wait collects for the roofline.
        g = torch.cuda.CUDAGraph()
        gp = torch.cuda.CUDAGraph() if not args.no_profile else g
        try:
            ctx.set_profiling(False)
            ctx.reset_stats()
            with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                async_call()
            graph_launches = ctx.stats()["kernel_launches"]
            if gp is not g:
                ctx.set_profiling(True)
                with torch.cuda.graph(gp, stream=stream, capture_error_mode="relaxed"):
                    async_call()
            with torch.cuda.stream(stream):
                g.replay()
                gp.replay()
            torch.cuda.synchronize()
            n_step = [0]

            def step():
                n_step[0] += 1
                (gp if n_step[0] == args.steps else g).replay()
        except Exception as ex:  # keep the run: eager calls instead
            print(f"bench: CUDA-graph capture failed ({ex}); timing eager calls", file=sys.stderr)
            torch.cuda.synchronize()
            ctx.close()
            ctx = Context(dev, stream)
            if sharded:
                ctx.comm_init_torch()
            args.graph = False
            graph_launches = None

    def barrier():
        if sharded:
            torch.distributed.barrier()

    clocks = ClockSampler(dev)
    ctx.reset_stats()
    if not args.no_profile and not args.graph:
        ctx.set_profiling(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks.stop()
    ms = e0.elapsed_time(e1)
    if sharded:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    stats = ctx.stats()
    if args.graph and not args.no_profile:
        ctx.wait()  # collects the captured events of the last replay
    prof = ctx.profile() if not args.no_profile else None
    psteps = 1 if args.graph else args.steps  # steps the profile covers
    ctx.set_profiling(False)
    ms_step = ms / args.steps
    value = F * args.steps / (ms * 1e-3) / 1e9   # one factorisation per step, whole job

    # ---- e2e: the literal C-ABI entry on pinned host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e and sharded:
        # the sharded entry from pinned host memory: H2D of the rank's columns, the
        # collective factorisation, D2H of its T columns and U / V rows
        Ah = torch.empty((lay["ncols"], m), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A_loc.t())
        Th = torch.empty_like(Ah)
        Uh = torch.empty((U_loc.shape[1], U_loc.shape[0]), dtype=torch.float64, pin_memory=True)
        Vh = torch.empty((n, lay["v1"] - lay["v0"]), dtype=torch.float64, pin_memory=True)

        def e2e_step():
            with torch.cuda.stream(stream):
                T_loc.copy_(Ah.t(), non_blocking=True)
                if trunc_k:
                    ctx.randutv_factor_dist_rank(T_loc, m, n, trunc_k, b, q, seed, Uk_local=U_loc, V_local=V_loc)
                else:
                    ctx.randutv_factor_dist(T_loc, m, n, b, q, seed, U_local=U_loc, V_local=V_loc)
                Th.copy_(T_loc.t(), non_blocking=True)
                Uh.copy_(U_loc.t(), non_blocking=True)
                Vh.copy_(V_loc.t(), non_blocking=True)
            stream.synchronize()

        e2e_step()
        e2e_steps = min(args.steps, 2)
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        dt = float(tt.item())
        bi = torch.tensor([8 * m * lay["ncols"]], device="cuda", dtype=torch.float64)
        bo = torch.tensor([8 * (m * lay["ncols"] + U_loc.numel() + V_loc.numel())],
                          device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(bi)
        torch.distributed.all_reduce(bo)
        e2e = {"value": F * e2e_steps / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(bi.item()),
               "d2h_bytes_per_step": int(bo.item()), "steps": e2e_steps, "ms_per_step": dt / e2e_steps * 1e3,
               "api": "randutv_factor_dist (pinned host shards)"}
    elif not args.no_e2e and trunc_k is None:
        # the literal C-ABI entry on pinned host buffers, copies inside the timed region
        Ah = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A.t())
        Uh = torch.empty((m, m), dtype=torch.float64, pin_memory=True)
        Th = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        Vh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        An, Un, Tn, Vn = Ah.numpy().T, Uh.numpy().T, Th.numpy().T, Vh.numpy().T
        del T, U, V  # make room for the library's host-staging buffers
        torch.cuda.empty_cache()
        randutv_factor(m, n, An, m, b, q, seed, Un, Tn, Vn)      # warm-up (allocates staging)
        e2e_steps = min(args.steps, 2)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            randutv_factor(m, n, An, m, b, q, seed, Un, Tn, Vn)
        dt = time.perf_counter() - t0
        e2e = {"value": F * e2e_steps / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * m * n,
               "d2h_bytes_per_step": 8 * (m * m + m * n + n * n), "steps": e2e_steps,
               "ms_per_step": dt / e2e_steps * 1e3, "api": "randutv_factor (literal entry, pinned host pointers)"}

    # ---- CPU baseline: the oracle on a bounded sample, rank 0, N = 1 only
    cpu = None
    if rank == 0 and ws == 1 and not sharded and not args.no_cpu_baseline:
        sm_, sn_ = sample_shape(args.config)
        A_host = np.asfortranarray(A[:sm_, :sn_].cpu().numpy())
        cpu = cpu_sample(args.config, A_host, seed)
        cpu = {k: v for k, v in cpu.items() if k not in ("seconds", "flops")}

    if rank == 0:
        peak, peak_src = fp64_peak()
        roof = None
        if prof and prof["dgemm"]["ms"] > 0:
            g = prof["dgemm"]
            # DGEMM launches of the main, V (and side) streams overlap: the time
            # the kernel ran is the UNION of their event spans (busy_ms); the
            # summed spans (ms) count concurrent launches twice
            busy = g.get("busy_ms") or g["ms"]
            # algorithmic GEMM flops: the model's flops of the
            # factorisation less the panel-QR leaf flops, per profiled step; the
            # launches' sum of 2MNK also counts non-algorithmic products (the
            # fused update's Z2^T W_U, the QR-internal W^T W) and is reported beside
            leaf_fl = prof.get("qr_leaf", {}).get("flops", 0.0) / psteps
            alg_fl = F / ws - leaf_fl   # sharded: this rank's share (the GEMM work splits by columns)
            ach = alg_fl / (busy / psteps * 1e-3) / 1e12
            ach_2mnk = g["flops"] / (busy * 1e-3) / 1e12
            traffic = None
            try:
                tr = json.load(open(NCU_TRAFFIC_FILE))
                if tr.get("config") == args.config:
                    traffic = tr.get("bytes_per_launch")
            except Exception:
                pass
            roof = {"bound": "tensor", "achieved": round(ach, 3), "peak": peak, "unit": "TFLOP/s",
                    "frac": round(ach / peak, 4), "traffic": traffic,
                    "kernel": "dgemm_kernel (mma.sync.m8n8k4.f64 / DMMA)",
                    "launches": g["launches"], "kernel_ms_per_step": round(busy / psteps, 3),
                    "kernel_share_of_step": round(busy / psteps / ms_step, 4),
                    "summed_launch_spans_ms_per_step": round(g["ms"] / psteps, 3),
                    "timing": "CUDA events around every launch inside the timed region; achieved = algorithmic "
                              "GEMM flops / union of the launch spans across streams",
                    "peak_source": peak_src,
                    "algorithmic": "SURVEY.md §8(d) M3 flops of the step less the panel-QR leaf flops (the DGEMM "
                                   "share of the model)",
                    "achieved_sum_2mnk": round(ach_2mnk, 3)}
            roof["other_kernels"] = {k: {"ms_per_step": v["ms"] / psteps, "launches": v["launches"]}
                                     for k, v in prof.items() if k != "dgemm"}
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_dict(args.config, ws, sharded),
                           **({"reorth": True, "note": "re-orthonormalised power steps; their QRs are not in flops_per_step"}
                              if args.reorth else {}),
                           **({"cuda_graph": "one captured RANDUTV_ASYNC factorisation replayed per step; the "
                                             "last step replays the capture that also records the per-launch "
                                             "profiling events (the roofline)"}
                              if args.graph else {})),
            "t_over_n3_x1e10": ms_step * 1e-3 / float(n) ** 3 * 1e10,
            "frac_of_fp64_peak": round(value / ws / 1e3 / peak, 4),   # of N x per-GPU peak
            "gpu_launches": stats["kernel_launches"] if graph_launches is None else graph_launches * args.steps,
            "gpu_launches_per_step": (stats["kernel_launches"] / args.steps) if graph_launches is None
            else graph_launches,
            "clocks": clocks.summary(),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if sharded:
        torch.distributed.destroy_process_group()
    return 0


def host_model(m, n, b, q, slots):
    """algorithmic PCIe bytes of the T-only host-streamed
    run -- the driver's panel access sequence replayed with no cache (the floor
    without reuse), LRU and Belady eviction (flops.host_stream_traffic)."""
    from paper_2002_06960_b200.flops import host_stream_traffic
    out = {}
    for pol in ("none", "lru", "belady"):
        h, d = host_stream_traffic(m, n, b, q, slots, pol)
        out[pol] = {"h2d_bytes": h, "d2h_bytes": d}
    return out


def run_host_streamed(args):
    """S12: randutv_factor_host from pinned host memory through a bounded device
    panel cache, reported like the paper's Table 1: compute time
    (the same factorisation resident in HBM), I/O time (summed H2D + D2H copy
    durations), real time, and their ratios."""
    import numpy as np
    import torch

    from paper_2002_06960_b200.flops import randutv_flops
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    from paper_2002_06960_b200.randutv import RANDUTV_NO_UV, Context, colmajor, pinned_colmajor

    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    m, n, b, q = cfg["m"], cfg["n"], cfg["b"], cfg["q"]
    if args.q is not None:
        q = args.q
    seed = 2000 + int(args.config[1:])
    uv = not args.no_uv
    F = randutv_flops(m, n, b, q, build_uv=uv)
    A = make_config_torch(args.config)
    A0 = pinned_colmajor(m, n)
    torch.from_numpy(A0.T).copy_(A.t())
    Ah = pinned_colmajor(m, n)
    U = pinned_colmajor(m, m) if uv else None
    V = pinned_colmajor(n, n) if uv else None
    stream = torch.cuda.Stream()
    ctx = Context(0, stream)
    # compute-only reference: the same factorisation resident in HBM
    with torch.cuda.stream(stream):
        Td = colmajor(m, n)
        Ud = colmajor(m, m) if uv else None
        Vd = colmajor(n, n) if uv else None
        ctx.randutv_factor_ex(A, b, q, seed, build_uv=uv, U=Ud, T=Td, V=Vd)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.randutv_factor_ex(A, b, q, seed, build_uv=uv, U=Ud, T=Td, V=Vd)
        e1.record(stream)
        torch.cuda.synchronize()
        comp_ms = e0.elapsed_time(e1)
    del A, Td, Ud, Vd
    torch.cuda.empty_cache()
    cache = int((args.cache_gib * 2**30) if args.cache_gib else 8 * m * n // 4)
    reps = []
    for it in range(max(args.warmup, 0) + args.steps):
        np.copyto(Ah, A0)
        _, _, rep = ctx.randutv_factor_host(Ah, b, q, seed, build_uv=uv, U=U, V=V, cache_bytes=cache)
        if it >= args.warmup:
            reps.append(rep)
    real = sum(r["wall_ms"] for r in reps) / len(reps)
    io = sum(r["h2d_ms"] + r["d2h_ms"] for r in reps) / len(reps)
    r0 = reps[-1]
    cfgd = config_dict(args.config, 1)
    if not uv:
        cfgd["workload"] = cfgd["workload"].replace("with U and V", "T only (no orthonormal matrices)")
    if args.q is not None and args.q != cfg["q"]:
        cfgd["workload"] = cfgd["workload"].replace(f"q={cfg['q']}", f"q={q}")
        cfgd["q"] = q
        cfgd["flops_per_step"] = F
    line = {"metric": METRIC, "value": round(F / (real * 1e-3) / 1e9, 2), "unit": "GFLOP/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(real, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(cfgd, mode="host-streamed", build_uv=uv, flops_per_step=F,
                           device_cache_bytes=cache, cache_slots=r0["cache_slots"]),
            "table1": {"computational_time_s": comp_ms * 1e-3, "io_time_s": io * 1e-3, "real_time_s": real * 1e-3,
                       "real_over_comp": real / comp_ms, "comp_over_io": comp_ms / io if io > 0 else None,
                       "h2d_bytes": r0["h2d_bytes"], "d2h_bytes": r0["d2h_bytes"],
                       "h2d_GBps": r0["h2d_bytes"] / (r0["h2d_ms"] * 1e-3) / 1e9 if r0["h2d_ms"] > 0 else None,
                       "cache_hits": r0["cache_hits"], "cache_misses": r0["cache_misses"],
                       "eviction": "lru" if (uv or os.environ.get("RUTV_HOST_EVICT") == "lru") else "belady",
                       "model": host_model(m, n, b, q, r0["cache_slots"]) if not uv else None},
            "t_over_n3_x1e10": real * 1e-3 / float(n) ** 3 * 1e10}
    print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def run_hqrrp(args):
    """HQRRP (A P = Q R, Sec. 2 of the paper) of the config's matrix with the
    config's b, Q built unless --no-uv; device-timed like the randUTV line.
    A separate workload, not the BASELINE metric."""
    import torch

    from paper_2002_06960_b200.flops import hqrrp_flops
    from paper_2002_06960_b200.inputs import CONFIGS, make_config_torch
    from paper_2002_06960_b200.randutv import Context, colmajor

    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    m, n, b = cfg["m"], cfg["n"], cfg["b"]
    seed = 2000 + int(args.config[1:])
    if args.mode == "host":
        return run_hqrrp_host(args, m, n, b, seed)
    bq = not args.no_uv
    F = hqrrp_flops(m, n, b, build_q=bq)
    A = make_config_torch(args.config)
    R = colmajor(m, n)
    stream = torch.cuda.Stream()
    ctx = Context(0, stream)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            R.copy_(A)
            ctx.randutv_hqrrp(R, b, seed, build_q=bq)
        torch.cuda.synchronize()
        tot = 0.0
        for it in range(args.steps):
            R.copy_(A)
            if it == args.steps - 1 and not args.no_profile:
                ctx.set_profiling(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.randutv_hqrrp(R, b, seed, build_q=bq)
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        prof = ctx.profile() if not args.no_profile else {}
    ms = tot / args.steps
    # PK_OTHER (the "fold_wait" slot of randUTV) holds the sketch CPQR here
    names = {"fold_wait": "cpqr_sketch"}
    kernels = {names.get(k, k): {"launches": v["launches"], "ms": round(v["ms"], 3)}
               for k, v in prof.items() if v["launches"]}
    line = {"metric": "HQRRP FP64 GFLOP/s", "value": round(F / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} matrix (m={m}, n={n}), HQRRP b={b}" + (", Q built" if bq else ", R only"),
                       "m": m, "n": n, "b": b, "flops_per_step": F, "algo": "hqrrp",
                       "l2": "inputs larger than L2; no flush" if 8 * m * n > 126e6 else "input fits in L2; no flush"},
            "kernels_last_step": kernels}
    print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def run_hqrrp_host(args, m, n, b, seed):
    """HQRRP_left from pinned host memory (Sec. 2.3), Table-1 style:
    compute time = the in-HBM right-looking HQRRP (R only) of the same matrix."""
    import numpy as np
    import torch

    from paper_2002_06960_b200.flops import hqrrp_flops
    from paper_2002_06960_b200.inputs import make_config_torch
    from paper_2002_06960_b200.randutv import Context, colmajor, pinned_colmajor

    A = make_config_torch(args.config)
    A0 = pinned_colmajor(m, n)
    torch.from_numpy(A0.T).copy_(A.t())
    stream = torch.cuda.Stream()
    ctx = Context(0, stream)
    with torch.cuda.stream(stream):
        R = colmajor(m, n)
        R.copy_(A)
        ctx.randutv_hqrrp(R, b, seed, build_q=False)
        R.copy_(A)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.randutv_hqrrp(R, b, seed, build_q=False)
        e1.record(stream)
        torch.cuda.synchronize()
        comp_ms = e0.elapsed_time(e1)
    del A, R
    torch.cuda.empty_cache()
    Ah = pinned_colmajor(m, n)
    reps = []
    for it in range(max(args.warmup, 0) + args.steps):
        np.copyto(Ah, A0)
        _, _, rep = ctx.randutv_hqrrp_host(Ah, b, seed)
        if it >= args.warmup:
            reps.append(rep)
    real = sum(r["wall_ms"] for r in reps) / len(reps)
    io = sum(r["h2d_ms"] for r in reps) / len(reps)
    r0 = reps[-1]
    F = hqrrp_flops(m, n, b, build_q=False)
    line = {"metric": "HQRRP FP64 GFLOP/s", "value": round(F / (real * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(real, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} matrix (m={m}, n={n}), HQRRP_left from pinned host memory, b={b}",
                       "m": m, "n": n, "b": b, "flops_per_step": F, "algo": "hqrrp", "mode": "host-streamed (left-looking)"},
            "table1": {"computational_time_s": comp_ms * 1e-3, "io_time_s": io * 1e-3, "real_time_s": real * 1e-3,
                       "real_over_comp": real / comp_ms, "h2d_bytes": r0["h2d_bytes"], "d2h_bytes": r0["d2h_bytes"],
                       "h2d_GBps": r0["h2d_bytes"] / (r0["h2d_ms"] * 1e-3) / 1e9 if r0["h2d_ms"] > 0 else None}}
    print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.algo == "hqrrp":
        return run_hqrrp(args)
    if args.mode == "host":
        return run_host_streamed(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
