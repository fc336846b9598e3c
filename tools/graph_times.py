#!/usr/bin/env python3
"""Per-call latency of small convolutions with and without HD_FLAG_GRAPH (CUDA-graph
replay of the pass launches), host wall clock over back-to-back calls + one sync."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2306_10016_b200 import hdconv as H  # noqa: E402

ctx = H.Context(0)
cases = [("config1 64 (*) 40", (64,), (40,), [{"m": 32}]),
         ("2-D 300x700 (*) 40x50", (300, 700), (40, 50), [{"m": 512, "C": 1, "S": 2}] * 2),
         ("3-D 20x30x40 (*) 5x6x7", (20, 30, 40), (5, 6, 7), [{"m": 16, "C": 2, "S": 2}] * 3)]
for name, sf, sg, axes in cases:
    f, g = synth.random_pair(1, sf, sg)
    fd, gd = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    out = {"case": name}
    for tag, flags in (("plain", 0), ("graph", H.HD_FLAG_GRAPH)):
        plan = H.Plan.make(len(sf), axes, flags=flags)
        h = ctx.conv(fd, gd, plan=plan)
        for _ in range(50):
            ctx.conv(fd, gd, plan=plan, h=h)
        torch.cuda.synchronize()
        n = 2000
        t = time.perf_counter()
        for _ in range(n):
            ctx.conv(fd, gd, plan=plan, h=h)
        torch.cuda.synchronize()
        out[tag + "_us_per_call"] = round((time.perf_counter() - t) / n * 1e6, 2)
    print(json.dumps(out), flush=True)
