#!/usr/bin/env python
"""Per-CUDA-source-line stall samples and shared-memory wavefronts of an ncu
report (run here, no GPU).  usage: python tools/ncu_lines.py REP [n] [kernel-substring]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
fname = ""
h = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        S = h.index("Warp Stall Sampling (All Samples)")
        W = h.index("L1 Wavefronts Shared")
        I = h.index("Instructions Executed")
        continue
    if h is None or len(r) <= S:
        continue
    if r[0]:
        line = (fname, int(r[0]))
        agg[line][3] = r[1]
        continue
    a = agg[line]
    a[0] += num(r[S])
    a[1] += num(r[W])
    a[2] += num(r[I])
tot = sum(a[0] for a in agg.values()) or 1
totw = sum(a[1] for a in agg.values())
print(f"total samples {tot:.0f}, shared wavefronts {totw:.0f}")
for (f, ln), (s, w, i, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{f}:{ln:<5d} samp={s:5.0f} ({100 * s / tot:4.1f}%) wav={w:9.0f} inst={i:9.0f}  {src.strip()[:80]}")
