#!/usr/bin/env python3
"""hd_conv2d_dist at world 1 on a 512-row f (config 3's rank share at N = 8) by nchunks:
the chunk launches' fixed costs without the exchanges.  usage: slab_chunks.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2306_10016_b200 import hdconv as H  # noqa: E402

ctx = H.Context(0)
ctx.dist_init()
Lf, Lg = [512, 4096], [255, 255]
f = torch.randn(Lf, dtype=torch.complex128, device="cuda")
g = torch.randn(Lg, dtype=torch.complex128, device="cuda")
plan = H.Plan.make(2, [{"m": 512, "S": 16}, {"m": 512, "S": 16}])
for nch in (1, 2, 4):
    h = ctx.conv2d_dist(f, g, Lf, plan=plan, nchunks=nch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ctx.conv2d_dist(f, g, Lf, plan=plan, nchunks=nch, h=h)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"nchunks": nch, "ms": round(e0.elapsed_time(e1) / 20, 4)}), flush=True)
