"""GPU parity of the q = 9 staged-engine layouts (hd_s512.cuh): the eight-warp W8
layout (setmaxnreg register hand-over, residue 8 as FFT-256 halves) and the nine-warp
layout, for the convolution pass and for the x passes.  The layout is chosen per
process (HD_S512_W8 bit mask: 1 x passes, 2 convolution pass), so every mask runs in a
subprocess of its own; each compares the CUDA result with the CPU oracle (relative L2
<= 1e-11, north_star) and checks which kernel shape ran (threads per CTA)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# y: 4000 + 300 - 1 = 4299 -> q = 9 at m = 512 (the staged convolution pass);
# x: 3900 + 250 - 1 = 4149 -> q = 9 (the staged x passes, f and g rows in one launch)
CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
import oracle, synth
from paper_2306_10016_b200 import hdconv as H
ctx = H.Context(0)
out = {}
for name, sf, sg in [("conv_y", (4000, 40), (300, 9)), ("x_passes", (30, 3900), (7, 250)),
                     ("both", (4000, 3900), (300, 250))]:
    f, g = synth.random_pair(%(seed)d, sf, sg)
    plan = H.Plan.make(2, [{"m": 512}, {"m": 512}])
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(), plan=plan)
    torch.cuda.synchronize()
    h = h.cpu().numpy()
    if name == "both":  # sampled outputs (the full direct sum is minutes on the host)
        idx = synth.sample_indices(h.shape, n_random=4096, seed=5, edge=8)
        want = oracle.multiconv_sampled([f], [g], idx)
        got = h[tuple(np.asarray(idx).T)]
        err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    else:
        err = float(oracle.rel_l2(h, oracle.conv(f, g)))
    out[name] = err
out["launches"] = ctx.engine_launches(H.HD_ENGINE_S512)
print(json.dumps(out))
"""


@pytest.mark.parametrize("mask", [0, 1, 2, 3])
def test_q9_layouts_match_oracle(mask):
    env = dict(os.environ, HD_S512_W8=str(mask))
    r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT, "seed": 9100 + mask}], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name in ("conv_y", "x_passes", "both"):
        assert res[name] < 1e-11, (mask, name, res)
    assert res["launches"] >= 9  # three staged passes per problem
