#!/usr/bin/env python3
"""Host vs device time of one config-3 step through hd_conv2d_dist at world 1 (and of
the single-GPU pipeline for comparison): is the slab path host-bound?"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2306_10016_b200 import hdconv as H  # noqa: E402

d = synth.config_inputs(3)
f = torch.from_numpy(d["f"][0]).cuda()
g = torch.from_numpy(d["g"][0]).cuda()
Lf = list(f.shape)
ctx = H.Context(0)
ctx.dist_init()
plan = H.Plan.make(2, [{"m": 512, "S": 16}, {"m": 512, "S": 16}])
sp = ctx.slab(H.HD_C128, Lf, list(g.shape), 0, plan)
h = torch.empty(sp.out_hi - sp.out_lo, Lf[1] + g.shape[1] - 1, dtype=torch.complex128, device="cuda")
hp = torch.empty_like(h)
for name, fn in [("slab", lambda: ctx.conv2d_dist(f, g, Lf, plan=plan, h=h)),
                 ("pipeline", lambda: ctx.conv(f, g, plan=plan, h=hp))]:
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    host = []
    e0.record()
    for _ in range(n):
        t = time.perf_counter()
        fn()
        host.append(time.perf_counter() - t)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: device {e0.elapsed_time(e1) / n:.3f} ms/step, host call {1e3 * sum(host) / n:.3f} ms "
          f"(max {1e3 * max(host):.3f})", flush=True)
