#!/usr/bin/env python3
"""Wall time of hd_tune (per-axis, the documented space) on BASELINE configs 3 and 5,
the chosen plans, their median times, and how many candidates were timed / pruned."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_10016_b200 import hdconv as H  # noqa: E402

ctx = H.Context(0)
for name, Lf, Lg, N in (("config3", [4096, 4096], [255, 255], 1), ("config5", [2048, 2048], [1024, 1536], 6),
                        ("config2", [8192], [3000], 1)):
    kw = dict(N=N, reps=3)
    if name == "config2":
        kw["batch"] = 4096
    t = time.perf_counter()
    p = ctx.tune(H.HD_C128, Lf, Lg, **kw)
    dt = time.perf_counter() - t
    log = ctx.hd_tune_log()
    pruned = sum(1 for _, s in log if math.isinf(s))
    print(json.dumps({"problem": name, "tune_seconds": dt, "plan": p.as_dict()["axis"], "median_ms": p.tuned_seconds * 1e3,
                      "log": len(log), "pruned": pruned}), flush=True)
