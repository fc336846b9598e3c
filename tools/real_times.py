#!/usr/bin/env python3
"""Per-pass times of hd_conv_real on BASELINE config 3's (real) image and kernel."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2306_10016_b200 import hdconv as H  # noqa: E402

d = synth.config_inputs(3)
f = torch.from_numpy(np.ascontiguousarray(d["f"][0].real)).cuda()
g = torch.from_numpy(np.ascontiguousarray(d["g"][0].real)).cuda()
ctx = H.Context(0)
Lz = [(f.shape[0] + 1) // 2, f.shape[1]]
plans = {"tuned": ctx.tune(H.HD_C128, Lz, list(g.shape), reps=3)}
for spec in sys.argv[1:]:
    plans[spec] = H.Plan.make(2, json.loads(spec))
for name, p in plans.items():
    h = ctx.conv_real(f, g, plan=p)
    torch.cuda.synchronize()
    ctx.profile_reset(); ctx.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ctx.conv_real(f, g, plan=p, h=h)
    e1.record(); torch.cuda.synchronize()
    ctx.profile_enable(False)
    prof = ctx.profile_read()
    print(json.dumps({"plan": name, "axes": [p.axis[i].m for i in range(2)], "step_ms": e0.elapsed_time(e1) / 20,
                      "passes": {k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items()}}))
