#!/usr/bin/env python3
"""Run a few steps of one BASELINE config through the C ABI with a fixed plan
(no tuning) -- the command profiled by ncu (tools/README in DESIGN.md)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2306_10016_b200 import hdconv as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--plan", default="", help="JSON list of per-axis dicts (m, C, S, D)")
ap.add_argument("--explicit", action="store_true")
a = ap.parse_args()
d = synth.config_inputs(a.config)
ctx = H.Context(0)
fd = [torch.from_numpy(x).cuda() for x in d["f"]]
gd = [torch.from_numpy(x).cuda() for x in d["g"]]
nd = d["ndim"]
plan = H.Plan.make(nd, json.loads(a.plan)) if a.plan else None
if d.get("plan") and plan is None:
    plan = H.Plan.make(nd, [d["plan"]])
for _ in range(a.steps):
    if a.explicit:
        ctx.hd_conv_explicit(fd, gd, plan=plan)
    elif len(fd) > 1:
        ctx.multiconv(fd, gd, plan=plan)
    else:
        ctx.conv(fd[0], gd[0], plan=plan, batch=(nd == 1 and d["batch"] > 1))
torch.cuda.synchronize()
print("ok launches", ctx.launch_count())
