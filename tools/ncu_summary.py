#!/usr/bin/env python
"""Summarise an ncu report (run here, no GPU): key metrics + hottest SASS lines.
usage: python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [n_hot]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n_hot = int(sys.argv[2]) if len(sys.argv) > 2 else 40
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "One or More Eligible", "Avg. Active Threads Per Warp"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in KEYS and d["Metric Name"] not in seen:
        seen.add(d["Metric Name"])
        print(f"{d['Metric Name']:<40} {d['Metric Value']:>14} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h, v = rr[0], rr[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg"):
        if k in h:
            print(f"{k:<40} {v[h.index(k)]:>14} {rr[1][h.index(k)]}")
    stall = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warp_latency_issue_stalled") or h[i].startswith("smsp__pcsamp_warps_issue_stalled")]
    tops = sorted(((float(x.replace(',', '')) if x.replace(',', '').replace('.', '').isdigit() else 0.0, n) for n, x in stall), reverse=True)[:10]
    for val, n in tops:
        print(f"  stall {n:<70} {val}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
if blocks:
    b = blocks[0]
    h = b[0]
    ix = {k: i for i, k in enumerate(h)}
    data = [r for r in b[1:] if len(r) == len(h)]
    samp = "Warp Stall Sampling (All Samples)"
    tot = sum(int(r[ix[samp]] or 0) for r in data)
    print(f"total stall samples {tot}")
    hot = sorted(data, key=lambda r: -int(r[ix[samp]] or 0))[:n_hot]
    for r in sorted(hot, key=lambda r: int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else 0):
        print(f"{r[ix['Address']][-5:]} {r[ix['Source']][:62]:<62} samp={r[ix[samp]]:>6} exec={r[ix['Instructions Executed']]}")
