#!/usr/bin/env python3
"""Device time of one rank's slab stages (hd_slab_stage, no exchange) at world sizes
1..8 on one GPU, config 3: what a rank computes per step at N GPUs (the exchanges
themselves need N GPUs).  Stage buffers are zero-filled -- timing only.
usage: slab_stage_times.py [--worlds 1,2,4,8] [--reps 20]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2306_10016_b200 import hdconv as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--nchunks", default="0", help="comma list of nchunks (0: the library default)")
a = ap.parse_args()
Lf, Lg = [4096, 4096], [255, 255]
dt = H.HD_C128
ctx = H.Context(0)
plan = H.Plan.make(2, [{"m": 512, "S": 16}, {"m": 512, "S": 16}])
import itertools  # noqa: E402
for world, nch in itertools.product([int(w) for w in a.worlds.split(",")], [int(c) for c in a.nchunks.split(",")]):
    sp = H.slab_plan(dt, Lf, Lg, world, 0, nch, plan)
    el = H.slab_buffer_elems(dt, sp, Lf, Lg)
    z = lambda n: torch.zeros(max(int(n), 1), dtype=torch.complex128, device="cuda")  # noqa: E731
    g = torch.zeros(Lg, dtype=torch.complex128, device="cuda")
    f = torch.zeros([sp.in_hi - sp.in_lo, Lf[1]], dtype=torch.complex128, device="cuda")
    h = torch.zeros([sp.out_hi - sp.out_lo, Lf[1] + Lg[1] - 1], dtype=torch.complex128, device="cuda")
    gt, x1, x2 = z(el["g"]), z(el["x1"]), z(el["x2"])
    stages = [(0, g, gt, None), (1, f, x1, None), (2, x1, x2, gt), (3, x2, h, None)]
    res = {}
    for st, inp, out, gtt in stages:
        for _ in range(3):
            ctx.slab_stage(dt, sp, Lf, Lg, st, inp, out, gt=gtt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            ctx.slab_stage(dt, sp, Lf, Lg, st, inp, out, gt=gtt)
        e1.record()
        torch.cuda.synchronize()
        res[f"stage{st}"] = round(e0.elapsed_time(e1) / a.reps, 4)
    res["sum_ms"] = round(sum(res.values()), 4)
    print(json.dumps({"world": world, "nchunks": sp.nchunks, "rows": sp.in_hi - sp.in_lo,
                      "cols": sp.spec_hi - sp.spec_lo, "ms": res}), flush=True)
