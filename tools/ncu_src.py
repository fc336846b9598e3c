#!/usr/bin/env python3
"""Stall samples and shared-memory wavefronts by SASS opcode (and the top
instructions) for one kernel of an ncu report's source page.
usage: ncu_src.py <report.ncu-rep> <kernel-substring> [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None:
        cur[2].append(r)
for name, hdr, data in blocks:
    if ksub not in name:
        continue
    idx = {h: j for j, h in enumerate(hdr)}
    num = lambda x: float(x) if x not in ("", None) else 0.0
    S = "Warp Stall Sampling (All Samples)"
    tot = sum(num(r[idx[S]]) for r in data)
    print(name, "samples", tot)
    c, ci, cw = Counter(), Counter(), Counter()
    for r in data:
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        c[op] += num(r[idx[S]])
        ci[op] += num(r[idx["Instructions Executed"]])
        cw[op] += num(r[idx["L1 Wavefronts Shared"]])
    for op, v in c.most_common(top):
        print(f"  {op:10s} stall {100 * v / tot:5.1f}%  warp-instr {ci[op]:.3e}  smem wavefronts {cw[op]:.3e}")
    break
