#!/usr/bin/env python3
"""Time a list of plans for one BASELINE config (CUDA events, per-pass profile).

    python tools/sweep.py --config 3 --plans '[[{"m":512,"S":1,"D":9},{"m":512,"C":2}], ...]'
    python tools/sweep.py --config 3 --tune
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2306_10016_b200 import hdconv as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--plans", default="[]")
ap.add_argument("--tune", action="store_true")
ap.add_argument("--default", action="store_true")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
d = synth.config_inputs(a.config)
nd = d["ndim"]
ctx = H.Context(0)
fd = [torch.from_numpy(x).cuda() for x in d["f"]]
gd = [torch.from_numpy(x).cuda() for x in d["g"]]
N = len(fd)
dt = H.HD_C128 if fd[0].dtype == torch.complex128 else H.HD_C64
Lf = list(d["f"][0].shape[-nd:])
Lg = list(d["g"][0].shape[-nd:])
Lout = [x + y - 1 for x, y in zip(Lf, Lg)]
nout = int(np.prod(Lout)) * d["batch"]
plans = [H.Plan.make(nd, p) for p in json.loads(a.plans)]
if a.default:
    plans.insert(0, H.hd_plan_default(dt, Lf, Lg, npairs=N))
if a.tune:
    plans.append(ctx.tune(dt, Lf, Lg, N=N, batch=d["batch"], reps=3))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run(p):
    if N > 1:
        ctx.multiconv(fd, gd, plan=p)
    else:
        ctx.conv(fd[0], gd[0], plan=p, batch=(nd == 1 and d["batch"] > 1))


for p in plans:
    try:
        run(p)
        run(p)
        torch.cuda.synchronize()
        ctx.profile_reset()
        ctx.profile_enable(True)
        e0.record()
        for _ in range(a.reps):
            run(p)
        e1.record()
        torch.cuda.synchronize()
        ctx.profile_enable(False)
        ms = e0.elapsed_time(e1) / a.reps
        prof = {k: round(v[0] / v[1], 4) for k, v in ctx.profile_read().items()}
        pc = H.hd_plan_complete(dt, Lf, Lg, H.Plan.from_buffer_copy(p), npairs=N)
        desc = [(x["m"], x["C"], x["S"], x["D"], x["threads"]) for x in pc.as_dict()["axis"]]
        print(json.dumps({"plan(m,C,S,D,threads)": desc, "ms": round(ms, 4),
                          "Gsamples/s": round(nout / ms / 1e6, 3), "passes_ms": prof}), flush=True)
    except Exception as ex:
        print(json.dumps({"plan": p.as_dict(), "error": str(ex)}), flush=True)
