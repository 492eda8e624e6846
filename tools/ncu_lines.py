#!/usr/bin/env python
"""Warp-stall samples per CUDA source line of an ncu report (joins the SASS
page's per-instruction samples with the cuda,sass listing's line mapping).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=30):
    sass = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    h = rows[1]
    ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    samples = {r[ai]: float(r[si] or 0) for r in rows[2:] if len(r) > si}
    both = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                          capture_output=True, text=True).stdout
    line, text = None, {}
    per = collections.Counter()
    for r in csv.reader(io.StringIO(both)):
        if len(r) < 4 or r[0] in ("File Path", "Function Name", "Line No"):
            continue
        if r[0]:
            line = int(r[0])
            text[line] = r[1]
        elif r[2] in samples and line is not None:
            per[line] += samples[r[2]]
    tot = sum(per.values()) or 1.0
    for ln, v in per.most_common(top):
        print(f"{100 * v / tot:5.1f}% {ln:5d}  {text[ln][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
