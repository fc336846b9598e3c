#!/usr/bin/env python3
"""Per-pass device times (CUDA events around each launch, hd_profile_*) of one
BASELINE config under several explicit plans.  Used to compare engines/plans
without the tuner.  usage: pass_times.py --config 3 --plans '[[{..},{..}], ...]'"""
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
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--plans", required=True, help="JSON list of plans (each a list of per-axis dicts)")
a = ap.parse_args()
d = synth.config_inputs(a.config)
ctx = H.Context(0)
fd = [torch.from_numpy(x).cuda() for x in d["f"]]
gd = [torch.from_numpy(x).cuda() for x in d["g"]]
nd = d["ndim"]


def step(plan):
    if len(fd) > 1:
        ctx.multiconv(fd, gd, plan=plan)
    else:
        ctx.conv(fd[0], gd[0], plan=plan, batch=(nd == 1 and d["batch"] > 1))


for axes in json.loads(a.plans):
    flags = 0
    if isinstance(axes, dict):
        flags = axes.get("flags", 0)
        axes = axes["axes"]
    plan = H.Plan.make(nd, axes, flags=flags)
    try:
        for _ in range(3):
            step(plan)
    except H.HDError as e:
        print(json.dumps({"plan": axes, "error": str(e)}), flush=True)
        continue
    torch.cuda.synchronize()
    ctx.profile_reset()
    e0 = [ctx.engine_launches(e) for e in range(5)]
    ctx.profile_enable(True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(a.steps):
        step(plan)
    s1.record()
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    prof = ctx.profile_read()
    eng = [(ctx.engine_launches(e) - e0[e]) // a.steps for e in range(5)]
    out = {"plan": axes, "flags": flags, "step_ms": s0.elapsed_time(s1) / a.steps,
           "engines": dict(zip(["generic", "s512", "s512_mconv", "s128", "s512c"], eng)),
           "passes": {k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items()}}
    print(json.dumps(out), flush=True)
