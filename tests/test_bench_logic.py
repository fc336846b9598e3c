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


class _Ax:
    def __init__(self, m, q, pf, pg, M1):
        self.m, self.q, self.p_f, self.p_g, self.M1 = m, q, pf, pg, M1


class _Plan:
    def __init__(self, axes):
        self.axis = axes


def test_conv_flops_config3(bench):
    # per line: (2N+1) q 5 m log2 m + 8 m q (p_f + p_g) N + 8 m q T + 6 m q N, lines = M1_x
    plan = _Plan([_Ax(512, 9, 8, 1, 4608), _Ax(512, 9, 8, 1, 4608)])
    fl = bench.conv_flops(2, 1, [4096, 4096], [255, 255], [4350, 4350], plan)
    m, q, T = 512, 9, 9
    per_line = 3 * q * 5 * m * 9 + 8 * m * q * 9 + 8 * m * q * T + 6 * m * q
    assert fl == pytest.approx(per_line * 4608)
    assert fl == pytest.approx(6.051594240e9)  # the bench line's alg_flops_per_launch


def test_fp64_peak_derivation(bench):
    assert bench.FP64_PEAK_TFLOPS == pytest.approx(2 * 64 * 148 * 1.965e9 / 1e12)
    assert np.isclose(bench.FP64_PEAK_TFLOPS, 37.22496)
