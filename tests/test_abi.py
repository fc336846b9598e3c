"""Host-side checks of the C ABI (no GPU needed): the library loads, exports every
symbol include/hdconv.h declares, computes plans as the paper defines them, and
refuses compute without a device (no CPU fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import build
    build.build()
    from paper_2306_10016_b200 import hdconv
    return hdconv


def test_exports_every_declared_symbol(H):
    hdr = open(os.path.join(ROOT, "include", "hdconv.h")).read()
    declared = set(re.findall(r"\b(hd_[a-z0-9_]+)\s*\(", hdr))
    declared -= {"hd_ctx"}
    assert declared, "no declarations parsed"
    lib = H.lib()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(H.EXPORTED) == declared


def test_abi_version(H):
    assert H.hd_abi_version() == 1


def test_plan_arithmetic_golden(H, golden):
    # p = ceil(L/m), q = ceil(M/m) (figure caption)
    d = golden("plan_examples.json")
    for c in d["cases"]:
        # a 1D problem whose f has length L and whose M is the case's M
        Lg = max(1, c["M"] - c["L"] + 1)
        p = H.Plan.make(1, [{"m": c["m"]}], flags=H.HD_FLAG_ALLOW_ALIAS)
        H.hd_plan_complete(H.HD_C128, [c["L"]], [Lg], p, M=[c["M"]])
        assert p.axis[0].p_f == c["p"] and p.axis[0].q == c["q"]
        assert p.axis[0].p_f * c["m"] == c["explicit"]
        assert p.axis[0].M1 == c["implicit"]


def test_config1_plan(H):
    p = H.Plan.make(1, [{"m": 32}])
    H.hd_plan_complete(H.HD_C128, [64], [40], p)
    a = p.axis[0]
    assert (a.m, a.p_f, a.p_g, a.q, a.M1, a.D) == (32, 2, 2, 4, 128, 4)


def test_plan_validation(H):
    with pytest.raises(H.HDError):  # m not a power of two
        H.hd_plan_complete(H.HD_C128, [10], [10], H.Plan.make(1, [{"m": 12}]))
    with pytest.raises(H.HDError):  # M < Lf + Lg - 1 would alias
        H.hd_plan_complete(H.HD_C128, [10], [10], H.Plan.make(1, [{"m": 4}]), M=[12])
    with pytest.raises(H.HDError):  # D > q
        H.hd_plan_complete(H.HD_C128, [10], [10], H.Plan.make(1, [{"m": 4, "D": 9}]))
    with pytest.raises(H.HDError):  # lines*D*m beyond shared memory
        H.hd_plan_complete(H.HD_C128, [4096], [4096], H.Plan.make(1, [{"m": 4096, "C": 4}]))
    with pytest.raises(H.HDError):  # tile width S must be a power of two <= 16
        H.hd_plan_complete(H.HD_C64, [8, 8, 8], [3, 3, 3],
                           H.Plan.make(3, [{"m": 8, "S": 3}, {"m": 8, "S": 1}, {"m": 8}]))
    with pytest.raises(H.HDError):  # threads must be a multiple of 32
        H.hd_plan_complete(H.HD_C128, [10], [10], H.Plan.make(1, [{"m": 4, "threads": 100}]))
    for Lf, Lg in [([0], [5]), ([5], [0]), ([4, 0], [3, 3]), ([-1], [2])]:  # empty / negative extents
        with pytest.raises(H.HDError):
            H.hd_plan_complete(H.HD_C128, Lf, Lg, H.Plan.make(len(Lf), [{"m": 4}] * len(Lf)))
        with pytest.raises(H.HDError):
            H.hd_plan_default(H.HD_C128, Lf, Lg)


def test_default_plans_are_admissible(H):
    cases = [(H.HD_C128, [64], [40], 1), (H.HD_C128, [8192], [3000], 1),
             (H.HD_C128, [4096, 4096], [255, 255], 1), (H.HD_C64, [512] * 3, [129] * 3, 1),
             (H.HD_C128, [2048, 2048], [1024, 1536], 6), (H.HD_C128, [1], [1], 1)]
    for dt, Lf, Lg, n in cases:
        p = H.hd_plan_default(dt, Lf, Lg, npairs=n)
        H.hd_plan_complete(dt, Lf, Lg, p, npairs=n)
        for i in range(len(Lf)):
            a = p.axis[i]
            assert a.M1 == a.q * a.m >= Lf[i] + Lg[i] - 1
            assert a.p_f == -(-Lf[i] // a.m) and a.p_g == -(-Lg[i] // a.m)
            assert 1 <= a.D <= a.q


@pytest.mark.parametrize("m", [2, 4, 8, 16, 32, 64, 128, 512, 1024, 4096])
def test_spectral_permutation_is_a_bijection(H, m):
    perm = H.hd_spectral_permutation(m)
    assert sorted(perm.tolist()) == list(range(m))


def test_no_cpu_fallback(H):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HDError) as e:
        H.Context(0)
    assert e.value.status == H.HD_ERR_CUDA


def test_window_modes_match_the_paper_formulas(H):
    """Output windows of the paper's 2-D listing (worked values
    SPEC.md:269-274): for L1 = 3, L2 = 5 (N = 7): full (0, 7), same_big (0, 5),
    same_small (1, 4), valid (ceil(7/5) - 1, ceil(7/3) + 1) = (1, 4)."""
    cases = {"full": (0, 7), "same_big": (0, 5), "same_small": (1, 4), "valid": (1, 4)}
    for mode, (v, v1) in cases.items():
        lo, n = H.window_for_mode(mode, [3, 3], [5, 5])
        assert lo == [v, v] and n == [v1 - v, v1 - v], mode
    # a 3-tap kernel over a 100-sample line: same_big keeps the first 100 outputs
    assert H.window_for_mode("same_big", [3], [100]) == ([0], [100])
    with pytest.raises(ValueError):
        H.window_for_mode("nope", [3], [5])


def test_filter_dictionary_matches_paper(H, golden):
    """hd_filter_kernel returns the eight kernels of the paper's image-filter listing
    (PAPER.md:1511-1520), in its dictionary order, with the listed scale factors."""
    import numpy as np
    d = golden("filter_kernels.json")
    assert H.FILTER_NAMES == d["order"]
    for i, name in enumerate(d["order"]):
        k = d["kernels"][name]
        ref = np.asarray(k["rows"], dtype=np.float64) * k["scale"][0] / k["scale"][1]
        got_name, w = H.filter_kernel(i)
        assert got_name == name
        assert w.shape == ref.shape and np.array_equal(w, ref)
    with pytest.raises(H.HDError):
        H.filter_kernel(8)


def test_default_plan_long_1d_lines(H):
    """Config 2's lines (8192 (*) 3000, c128): the default plan is m = 4096 with every
    residue in one pass (q = 3, the one-CTA-per-line engine hd_s4096r.cuh), p_f = 2,
    p_g = 1 (PAPER.md:564-567 at m = 4096, M = 11191); lines of q > 4 at m = 4096 keep
    the cost model's pick."""
    p = H.hd_plan_complete(H.HD_C128, [8192], [3000], H.hd_plan_default(H.HD_C128, [8192], [3000]))
    a = p.axis[0]
    assert (a.m, a.q, a.D, a.p_f, a.p_g, a.M1) == (4096, 3, 3, 2, 1, 12288)
    p = H.hd_plan_complete(H.HD_C128, [30000], [3000], H.hd_plan_default(H.HD_C128, [30000], [3000]))
    assert p.axis[0].m != 4096 or p.axis[0].q <= 4
