#!/usr/bin/env python
"""Stall breakdown of an ncu report: totals per reason and per opcode (SASS source page).

    python tools/ncu_stalls.py gpurun_out/prof_skinny.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

KS = ['stall_wait', 'stall_math', 'stall_long_sb', 'stall_barrier', 'stall_short_sb', 'stall_selected',
      'stall_not_selected', 'stall_branch_resolving', 'stall_dispatch', 'stall_no_inst', 'stall_mio', 'stall_lg']


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    for w in ['Kernel Name', 'Grid Size', 'Block Size', 'gpu__time_duration.sum',
              'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
              'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'sm__warps_active.avg.pct_of_peak_sustained_active',
              'dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
              'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum']:
        if w in h:
            print(f"{w:80s} {v[h.index(w)]}")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    isrc, iall = h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
    ix = {k: h.index(k) for k in KS if k in h}
    # multi-kernel reports repeat the header per kernel: keep the first kernel's rows
    data = []
    for r in rows[2:]:
        if len(r) > iall and r[iall] == 'Warp Stall Sampling (All Samples)':
            break
        data.append(r)

    def g(r, k):
        try:
            return int(r[ix[k]] or 0)
        except (ValueError, IndexError, KeyError):
            return 0
    T = sum(int(r[iall] or 0) for r in data if len(r) > iall)
    tot = {k: sum(g(r, k) for r in data) for k in ix}
    print("samples", T, " ".join(f"{k[6:]}={v / T:.1%}" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
    grp, grpw = collections.Counter(), collections.defaultdict(collections.Counter)
    for r in data:
        if len(r) <= iall:
            continue
        op = r[isrc].strip().split()
        if not op:
            continue
        o = (op[1] if op[0].startswith('@') else op[0]).split('.')[0]
        grp[o] += int(r[iall] or 0)
        for k in ix:
            grpw[o][k] += g(r, k)
    for o, s in grp.most_common(12):
        print(f"  {o:10s} {s / T:6.1%}", ", ".join(f"{k[6:]}={n}" for k, n in grpw[o].most_common(3)))


if __name__ == "__main__":
    main(sys.argv[1])
