#!/usr/bin/env python
"""Summarise ncu output into profiles/: launch-list shares and the top-kernel metrics.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/ncu_launches_r01.txt
    python tools/ncu_summary.py full gpurun_out/prof_dgemm_nt.ncu-rep > profiles/ncu_dgemm_r01.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("(anonymous namespace)::", "").replace("rutv::", "").replace("unnamed>::", "")
    m = re.match(r"void\s+(\w+)(<.*>)?", name)
    base = m.group(1) if m else name
    if base == "dgemm_kernel" and m and m.group(2):
        t = m.group(2)
        cfg = "128x64" if "128, 64" in t else ("128x128" if "128, 128" in t else "")
        tr = re.search(r">\s*,\s*(\d|true|false)\s*,\s*(\d|true|false)", t)
        op = ""
        if tr:
            op = ("T" if tr.group(1) in ("1", "true") else "N") + ("T" if tr.group(2) in ("1", "true") else "N")
        return f"dgemm_kernel[{cfg},{op}]"
    return base


def launches(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    mi = hdr.index("Metric Name")
    vi = hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit]
        us = v * scale
        k = short(r[ki])
        tot[k] += us
        cnt[k] += 1
    T = sum(tot.values())
    print("# ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:4rutv")
    print("#   (librandutv kernels only; cold-cache, serialised: compare SHARES)")
    print("# command: python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile (c3, one full step)")
    print(f"# launches profiled: {sum(cnt.values())}, summed kernel time {T/1000:.2f} ms")
    print(f"{'kernel':40s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, v in tot.most_common():
        print(f"{k:40s} {cnt[k]:8d} {v/1000:10.3f} {v/T:7.1%}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "sm__cycles_elapsed.avg.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
    for r in rows[2:]:
        print("# ncu --set full --clock-control none, one launch")
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                print(f"{w:80s} {r[i]:>24s} {units[i]}")
        st = sorted(((float(r[i]) if r[i] else 0.0, hdr[i]) for i in stall), reverse=True)[:8]
        print("# top warp stall reasons (cycles per issued instruction)")
        for v, h in st:
            print(f"  {h.replace('smsp__average_warp_latency_issue_stalled_', ''):60s} {v:8.3f}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
