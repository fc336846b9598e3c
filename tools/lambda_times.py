#!/usr/bin/env python3
"""Device time of the row-f1 path (hd_conv1d_lambda, Lambda > 1 residue matching) on
config 2's pairs for several (m, Lambda), next to the Lambda = 1 pipeline (hd_conv1d
with the default plan).  usage: lambda_times.py [--steps 10]"""
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
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
d = synth.config_inputs(2)
f, g = torch.from_numpy(d["f"][0]).cuda(), torch.from_numpy(d["g"][0]).cuda()
if f.shape[-1] > g.shape[-1]:
    f, g = g, f
ctx = H.Context(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


print(json.dumps({"lambda1_default_plan_ms": round(timeit(lambda: ctx.conv(f, g, batch=True)), 4),
                  "shape": [list(f.shape), list(g.shape)]}), flush=True)
for m, lam in [(1024, 1), (512, 2), (256, 4), (128, 8), (512, 4), (256, 8), (1024, 2), (512, 8)]:
    try:
        ms = timeit(lambda: ctx.conv1d_lambda(f, g, m, lam))
        print(json.dumps({"m": m, "Lambda": lam, "ms": round(ms, 4)}), flush=True)
    except H.HDError as e:
        print(json.dumps({"m": m, "Lambda": lam, "error": str(e)}), flush=True)
