#!/usr/bin/env python3
"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump per CUDA
source line: share of warp-stall samples and of executed instructions."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
stall = defaultdict(float)
inst = defaultdict(float)
text = {}
cur = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iI = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        text[cur] = r[1]
    if cur is None:
        continue
    try:
        stall[cur] += float(r[iS] or 0)
        inst[cur] += float(r[iI] or 0)
    except ValueError:
        pass
ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
for ln in sorted(stall, key=lambda k: -stall[k])[:top]:
    print(f"{100 * stall[ln] / ts:5.1f}% stall {100 * inst[ln] / ti:5.1f}% inst  {ln[0][:12]}:{ln[1]:<5d} {text.get(ln, '').strip()[:90]}")
