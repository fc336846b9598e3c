"""Host logic of bench.py (CPU): the algorithmic byte and flop counts the roofline
divides by (the figures DESIGN.md section 6 quotes for config 3)."""
import importlib.util
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_alg_bytes_config3(bench):
    Lf, Lg, Lout = [4096, 4096], [255, 255], [4350, 4350]
    ab = bench.alg_bytes(2, 1, Lf, Lg, Lout, 16)
    # each pass reads its inputs once and writes its outputs once (16 B per element)
    assert ab["fwd_x_f"] == 16 * (4096 * 4096 + 4096 * 4350)
    assert ab["fwd_x_g"] == 16 * (255 * 255 + 255 * 4350)
    assert ab["conv_y"] == 16 * ((4096 + 255) * 4350 + 4350 * 4350)
    assert ab["inv_x"] == 16 * 2 * 4350 * 4350
    assert sum(ab.values()) == 1_783_415_056


def test_alg_bytes_1d_3d_and_pairs(bench):
    ab1 = bench.alg_bytes(1, 1, [8192], [3000], [11191], 16, batch=4096)
    assert ab1 == {"conv1d": 4096 * 16 * (8192 + 3000 + 11191)}
    ab3 = bench.alg_bytes(3, 1, [512] * 3, [129] * 3, [640] * 3, 8)
    assert ab3["inv_y"] == ab3["inv_x"] == 8 * 2 * 640 ** 3
    assert ab3["fwd_y_f"] == 8 * (512 * 512 * 640 + 512 * 640 * 640)
    # N pairs: the forward inputs scale with N, the output does not
    ab5 = bench.alg_bytes(2, 6, [2048, 2048], [1024, 1536], [3071, 3583], 16)
    assert ab5["inv_x"] == 16 * 2 * 3071 * 3583
    assert ab5["fwd_x_f"] == 16 * 6 * (2048 * 2048 + 2048 * 3583)


def test_conv_flops_plan_independent(bench):
    """(2N+1) x 5 M log2 M + 6 M N per line at M = L_out, lines = L_out of the other axes
    (no naive fold/unfold, no padded M1 -- a worse plan cannot raise it)."""
    fl = bench.conv_flops(2, 1, [4096, 4096], [255, 255], [4350, 4350])
    per_line = 3 * 5 * 4350 * np.log2(4350) + 6 * 4350
    assert fl == pytest.approx(per_line * 4350)
    assert fl == pytest.approx(3.5445e9, rel=1e-4)
    # multiconv: 13 transforms per line for N = 6
    fl5 = bench.conv_flops(2, 6, [2048, 2048], [1024, 1536], [3071, 3583])
    assert fl5 == pytest.approx((13 * 5 * 3071 * np.log2(3071) + 36 * 3071) * 3583)


def test_fp64_peak_source(bench):
    tf, src = bench.fp64_peak()
    assert 10.0 < tf < 80.0
    assert src.startswith("measured") or src.startswith("derived")


def test_bench_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (torch.distributed.run,
    127.0.0.1); --dry-run exercises the launch with gloo and no GPU work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2


def test_bench_refuses_mismatched_world():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--dry-run"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)


def test_auto_mode_is_strong_for_one_problem(bench):
    """--mode auto at N > 1: the BASELINE configs run one problem over all ranks (2-D /
    3-D by slabs, the 1-D batch by pairs); one GPU keeps the single-GPU pipeline."""
    assert bench.pick_mode(1, 2, 1, 1) == "independent"
    assert bench.pick_mode(8, 2, 1, 1) == "slab"      # config 3
    assert bench.pick_mode(8, 3, 1, 1) == "slab"      # config 4
    assert bench.pick_mode(8, 1, 1, 4096) == "batch"  # config 2
    assert bench.pick_mode(8, 2, 6, 1) == "independent"  # config 5 (multi-pair): weak
    assert bench.pick_mode(2, 1, 1, 1) == "independent"
