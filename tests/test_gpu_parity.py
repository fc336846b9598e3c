"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Tolerance (north_star): relative L2 <= 1e-11 for complex128 and
<= 1e-5 for complex64.  Run with -m gpu on a B200."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.complex128: 1e-11, np.complex64: 1e-5}


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import hdconv
    return hdconv


@pytest.fixture(scope="module")
def ctx(H):
    c = H.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# ---------------------------------------------------------------- residue routines
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("m", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_fft_m_vs_naive_dft(ctx, H, dtype, m):
    # U1: q = 1, L = m: the residue transform is the size-m DFT
    x = synth.random_pair(m, (3, m), (1,))[0].astype(dtype)
    X = host(ctx.hd_forward_residues(dev(x), m, 1))
    perm = H.hd_spectral_permutation(m)
    for l in range(3):
        ref = oracle.dft(x[l], m, +1)
        got = np.empty(m, complex)
        got[perm] = X[l]
        assert oracle.rel_l2(got, ref) < TOL[dtype] / 10


@pytest.mark.parametrize("L,m,q", [(3, 2, 2), (13, 4, 5), (100, 16, 9), (255, 512, 9),
                                   (4096, 512, 9), (3000, 1024, 11), (129, 128, 5),
                                   (1000, 64, 17), (64, 32, 4), (5, 8, 1)])
def test_residue_blocks_vs_dft(ctx, H, L, m, q):
    # U2: block r equals DFT_{qm}(x padded)[q l + r]
    x = synth.random_pair(L + 7 * m, (2, L), (1,))[0]
    X = host(ctx.hd_forward_residues(dev(x), m, q))
    perm = H.hd_spectral_permutation(m)
    for l in range(2):
        full = oracle.dft(x[l], q * m, +1)
        for r in range(q):
            got = np.empty(m, complex)
            got[perm] = X[l, r * m:(r + 1) * m]
            assert oracle.rel_l2(got, full[r::q]) < 1e-12


@pytest.mark.parametrize("L,m,q", [(3, 2, 2), (100, 16, 9), (4096, 512, 9), (129, 128, 5)])
def test_round_trip(ctx, L, m, q):
    # U3: backward(forward(x)) = q m x
    x = synth.random_pair(L, (2, L), (1,))[0]
    X = ctx.hd_forward_residues(dev(x), m, q)
    y = host(ctx.hd_backward_residues(X, m, q, L)) / (q * m)
    assert oracle.rel_l2(y, x) < 1e-13


def test_spec_worked_residue_example(ctx, H, golden):
    d = golden("residue_forward.json")
    X = host(ctx.hd_forward_residues(dev(np.array([d["x"]], complex)), d["m"], d["q"]))
    perm = H.hd_spectral_permutation(d["m"])
    for r in (0, 1):
        got = np.empty(2, complex)
        got[perm] = X[0, 2 * r:2 * r + 2]
        want = np.array([complex(a, b) for a, b in d[f"r{r}"]])
        assert np.allclose(got, want, atol=1e-13)


# ---------------------------------------------------------------- 1D
def test_worked_example(ctx, H, golden):
    d = golden("worked_example_1d.json")
    for m in (2, 4, 8):
        h = host(ctx.conv(dev(np.array(d["f"], complex)), dev(np.array(d["g"], complex)),
                          plan=H.Plan.make(1, [{"m": m}])))
        assert np.allclose(h, d["h"], atol=1e-13)


def test_alias_fold(ctx, H, golden):
    d = golden("alias_fold_1d.json")
    p = H.Plan.make(1, [{"m": 2}], flags=H.HD_FLAG_ALLOW_ALIAS)
    h = host(ctx.conv(dev(np.array(d["f"], complex)), dev(np.array(d["g"], complex)),
                      M=[d["M"]], plan=p))
    assert np.allclose(h, d["h"], atol=1e-13)


def test_config1(ctx, H):
    d = synth.config_inputs(1)
    f, g = d["f"][0], d["g"][0]
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(1, [{"m": 32, "D": 4}])))
    assert h.shape == (103,)
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11


def test_random_1d_sweep(ctx, H):
    # randomised small problems, every admissible plan shape (SPEC.md:202 style)
    s = synth.Stream(99)
    for case in range(60):
        Lf = 1 + int(s.uniform(1)[0] * 64)
        Lg = 1 + int(s.uniform(1)[0] * 64)
        f, g = synth.random_pair(1000 + case, (Lf,), (Lg,))
        ref = oracle.conv(f, g)
        m = 2 ** (1 + case % 7)
        q = -(-(Lf + Lg - 1) // m)
        D = 1 + case % q
        C = 1 << (case % 3)
        h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(1, [{"m": m, "D": D, "C": C}])))
        assert oracle.rel_l2(h, ref) < 1e-11, (Lf, Lg, m, D, C)


@pytest.mark.parametrize("C,D", [(1, 0), (2, 3), (4, 1)])
def test_batched_1d(ctx, H, C, D):
    f, g = synth.random_pair(5, (7, 300), (7, 77))
    h = host(ctx.conv(dev(f), dev(g), batch=True,
                      plan=H.Plan.make(1, [{"m": 64, "C": C, "D": D}])))
    assert oracle.rel_l2(h, oracle.conv_batch(f, g)) < 1e-11
    # shared g
    hs = host(ctx.conv(dev(f), dev(g[0]), batch=True, shared_g=True))
    ref = np.stack([oracle.conv(f[b], g[0]) for b in range(7)])
    assert oracle.rel_l2(hs, ref) < 1e-11


def test_padding_monotonicity(ctx, H):
    # any M >= L_out gives the same first L_out outputs
    f, g = synth.random_pair(8, (37,), (21,))
    ref = oracle.conv(f, g)
    for M in (57, 58, 64, 100, 200):
        h = host(ctx.conv(dev(f), dev(g), M=[M], plan=H.Plan.make(1, [{"m": 8}])))
        assert oracle.rel_l2(h, ref) < 1e-11


def test_integer_exactness(ctx):
    f, g = synth.integer_pair(4, (500,), (300,))
    h = host(ctx.conv(dev(f), dev(g)))
    ref = oracle.conv(f, g)
    assert np.array_equal(np.round(h.real), ref.real) and np.array_equal(np.round(h.imag), ref.imag)
    assert np.max(np.abs(h - ref)) < 1e-9


def test_c64_1d(ctx):
    f, g = synth.random_pair(6, (1000,), (333,))
    h = host(ctx.conv(dev(f.astype(np.complex64)), dev(g.astype(np.complex64))))
    ref = oracle.conv(f.astype(np.complex64), g.astype(np.complex64))
    assert oracle.rel_l2(h, ref) < 1e-5


# ---------------------------------------------------------------- 2D / 3D / multiconv
PLANS_2D = [None,
            [{"m": 8, "S": 1, "D": 0}, {"m": 16, "C": 1, "D": 0}],
            [{"m": 16, "S": 2, "D": 2}, {"m": 8, "C": 2, "D": 3}],
            [{"m": 32, "S": 4, "D": 1}, {"m": 64, "C": 4, "D": 1}],
            [{"m": 4, "S": 8, "D": 5}, {"m": 4, "C": 8, "D": 2}]]


@pytest.mark.parametrize("pi", range(len(PLANS_2D)))
def test_2d_plans(ctx, H, pi):
    f, g = synth.random_pair(20 + pi, (45, 70), (13, 9))
    ref = oracle.conv(f, g)
    plan = None if PLANS_2D[pi] is None else H.Plan.make(2, PLANS_2D[pi])
    h = host(ctx.conv(dev(f), dev(g), plan=plan))
    assert oracle.rel_l2(h, ref) < 1e-11


def test_2d_batched_and_swapped(ctx):
    f, g = synth.random_pair(30, (3, 20, 33), (3, 41, 7))  # g longer on axis 0
    h = host(ctx.conv(dev(f), dev(g), batch=True))
    ref = np.stack([oracle.conv(f[b], g[b]) for b in range(3)])
    assert oracle.rel_l2(h, ref) < 1e-11


def test_2d_separability_and_delta(ctx):
    s = synth.Stream(31)
    a, b, c, d = (s.complex_uniform((n,)) for n in (30, 25, 7, 12))
    h = host(ctx.conv(dev(np.outer(a, b)), dev(np.outer(c, d))))
    assert oracle.rel_l2(h, np.outer(np.convolve(a, c), np.convolve(b, d))) < 1e-11
    g = s.complex_uniform((17, 19))
    delta = np.zeros((2, 3), complex)
    delta[1, 2] = 1
    h2 = host(ctx.conv(dev(delta), dev(g)))
    assert np.allclose(h2[1:, 2:], g, atol=1e-13) and np.max(np.abs(h2[0])) < 1e-13


def test_2d_c64(ctx):
    f, g = synth.random_pair(32, (100, 90), (20, 31), dtype=np.complex64)
    h = host(ctx.conv(dev(f), dev(g)))
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-5


PLANS_3D = [None,
            [{"m": 8, "S": 2, "D": 0}, {"m": 4, "S": 2, "D": 3}, {"m": 16, "C": 2, "D": 0}],
            [{"m": 16, "S": 1, "D": 1}, {"m": 8, "S": 1, "D": 0}, {"m": 8, "C": 4, "D": 2}],
            [{"m": 4, "S": 4, "D": 2}, {"m": 16, "S": 4, "D": 1}, {"m": 4, "C": 1, "D": 0}]]


@pytest.mark.parametrize("pi", range(len(PLANS_3D)))
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_3d_plans(ctx, H, pi, dtype):
    f, g = synth.random_pair(40 + pi, (19, 14, 23), (6, 9, 4), dtype=dtype)
    ref = oracle.conv(f, g)
    plan = None if PLANS_3D[pi] is None else H.Plan.make(3, PLANS_3D[pi])
    h = host(ctx.conv(dev(f), dev(g), plan=plan))
    assert oracle.rel_l2(h, ref) < TOL[dtype]


def test_multiconv(ctx, H):
    s = synth.Stream(50)
    fs = [s.complex_uniform((30, 41)) for _ in range(5)]
    gs = [s.complex_uniform((12, 23)) for _ in range(5)]
    ref = oracle.multiconv(fs, gs)
    h = host(ctx.multiconv([dev(a) for a in fs], [dev(a) for a in gs]))
    assert oracle.rel_l2(h, ref) < 1e-11
    p = H.Plan.make(2, [{"m": 8, "S": 2, "D": 2}, {"m": 16, "C": 2, "D": 1}])
    h = host(ctx.multiconv([dev(a) for a in fs], [dev(a) for a in gs], plan=p))
    assert oracle.rel_l2(h, ref) < 1e-11
    f1 = [s.complex_uniform((50,)) for _ in range(3)]
    g1 = [s.complex_uniform((20,)) for _ in range(3)]
    h1 = host(ctx.multiconv([dev(a) for a in f1], [dev(a) for a in g1]))
    assert oracle.rel_l2(h1, oracle.multiconv(f1, g1)) < 1e-11
    f3 = [s.complex_uniform((7, 8, 9)) for _ in range(2)]
    g3 = [s.complex_uniform((3, 4, 5)) for _ in range(2)]
    h3 = host(ctx.multiconv([dev(a) for a in f3], [dev(a) for a in g3]))
    assert oracle.rel_l2(h3, oracle.multiconv(f3, g3)) < 1e-11


def test_explicit_variant(ctx):
    f, g = synth.random_pair(60, (40, 33), (11, 20))
    h = host(ctx.hd_conv_explicit([dev(f)], [dev(g)]))
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11
    f1, g1 = synth.random_pair(61, (300,), (45,))
    h1 = host(ctx.hd_conv_explicit([dev(f1)], [dev(g1)]))
    assert oracle.rel_l2(h1, oracle.conv(f1, g1)) < 1e-11


def test_host_entry_point(ctx):
    f, g = synth.random_pair(70, (64, 50), (10, 12))
    h = np.zeros((73, 61), complex)
    ctx.hd_conv_host([f], [g], h, ndim=2)
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11


def test_host_async_pipeline(ctx):
    """hd_conv_host_async: five calls in flight over the three context slots (copy-in
    of call k+2 | convolution k+1 | copy-out k), different inputs, sizes and output buffers;
    every result checked after one hd_host_sync."""
    shapes = [((64, 50), (10, 12)), ((40, 33), (7, 9)), ((64, 50), (10, 12)), ((90, 20), (3, 31)),
              ((64, 50), (10, 12))]
    torch_ = pytest.importorskip("torch")
    jobs = []
    for i, (sf, sg) in enumerate(shapes):
        f, g = synth.random_pair(700 + i, sf, sg)
        ft, gt = torch_.from_numpy(f).pin_memory(), torch_.from_numpy(g).pin_memory()
        h = torch_.zeros([a + b - 1 for a, b in zip(sf, sg)], dtype=torch_.complex128).pin_memory()
        ctx.hd_conv_host_async([ft], [gt], h, ndim=2)
        jobs.append((f, g, ft, gt, h))
    ctx.host_sync()
    for f, g, _, _, h in jobs:
        assert oracle.rel_l2(h.numpy(), oracle.conv(f, g)) < 1e-11


def test_host_async_mixed_with_other_entries(H):
    """The async slots survive the other host/explicit entry points resizing their
    buffers, and a context with live slots closes cleanly (own context)."""
    torch_ = pytest.importorskip("torch")
    c = H.Context(0)
    f, g = synth.random_pair(720, (64, 50), (10, 12))
    ft, gt = torch_.from_numpy(f).pin_memory(), torch_.from_numpy(g).pin_memory()
    ref = oracle.conv(f, g)
    h1 = torch_.zeros(ref.shape, dtype=torch_.complex128).pin_memory()
    c.hd_conv_host_async([ft], [gt], h1, ndim=2)
    c.host_sync()
    fb, gb = synth.random_pair(721, (300, 200), (40, 30))
    hb = c.hd_conv_explicit([dev(fb)], [dev(gb)])   # grows the context's scratch
    hh = np.zeros((339, 229), complex)
    c.hd_conv_host([fb], [gb], hh, ndim=2)
    h2 = torch_.zeros(ref.shape, dtype=torch_.complex128).pin_memory()
    c.hd_conv_host_async([ft], [gt], h2, ndim=2)
    c.host_sync()
    assert oracle.rel_l2(h1.numpy(), ref) < 1e-11 and oracle.rel_l2(h2.numpy(), ref) < 1e-11
    refb = oracle.conv(fb, gb)
    assert oracle.rel_l2(host(hb), refb) < 1e-11 and oracle.rel_l2(hh, refb) < 1e-11
    c.close()


# ---------------------------------------------------------------- output windows (f3)
@pytest.mark.parametrize("case", [
    ("1d", (300,), (70,), (5,), (300,), None),
    ("2d-staged", (900, 700), (200, 90), (13, 77), (850, 600), None),
    ("2d-staged-mode", (600, 520), (31, 17), None, None, "same_big"),
    ("2d-generic", (300, 260), (31, 17), (3, 1), (320, 250), "generic"),
    ("2d-small-mode", (64, 50), (10, 12), None, None, "same_small"),
])
def test_output_window(ctx, H, case):
    """hd_conv_window: every output inside the window equals the oracle's full
    convolution at the same index (PAPER.md:1482-1489 modes are windows)."""
    name, sf, sg, lo, n, mode = case
    f, g = synth.random_pair(750 + len(name), sf, sg)
    if mode in ("same_big", "same_small"):
        lo, n = H.window_for_mode(mode, list(sf), list(sg))
    nd = len(sf)
    flags = H.HD_FLAG_GENERIC_FFT if mode == "generic" else 0
    m = 512 if "staged" in name else 64
    plan = H.Plan.make(nd, [{"m": m, "C": 1, "S": 2}] * nd, flags=flags)
    h = host(ctx.conv_window([dev(f)], [dev(g)], lo, n, plan=plan))
    full = oracle.conv(f, g)
    ref = full[tuple(slice(a, a + b) for a, b in zip(lo, n))]
    assert h.shape == ref.shape and oracle.rel_l2(h, ref) < 1e-11


def test_output_window_3d_c64_and_multiconv(ctx, H):
    f, g = synth.random_pair(760, (20, 18, 30), (5, 7, 4), dtype=np.complex64)
    lo, n = [2, 0, 9], [15, 20, 20]
    h = host(ctx.conv_window([dev(f)], [dev(g)], lo, n))
    full = oracle.conv(f, g)
    ref = full[2:17, 0:20, 9:29]
    assert oracle.rel_l2(h, ref) < 1e-5
    fs, gs = zip(*[synth.random_pair(770 + k, (700, 130), (520, 20)) for k in range(3)])
    lo, n = [100, 7], [1000, 120]
    plan = H.Plan.make(2, [{"m": 512, "C": 1, "S": 2}] * 2)
    h = host(ctx.conv_window([dev(x) for x in fs], [dev(x) for x in gs], lo, n, plan=plan))
    ref = oracle.multiconv(list(fs), list(gs))[100:1100, 7:127]
    assert oracle.rel_l2(h, ref) < 1e-11


def test_output_window_rejects_outside(ctx, H):
    f, g = synth.random_pair(780, (30, 20), (5, 5))
    with pytest.raises(H.HDError):
        ctx.conv_window([dev(f)], [dev(g)], [0, 0], [35, 25])


# ---------------------------------------------------------------- real inputs (f2)
@pytest.mark.parametrize("sf,sg,m", [((101,), (40,), 32), ((1,), (7,), 4), ((900, 700), (200, 90), 512),
                                     ((301, 260), (31, 17), 64), ((20, 18, 30), (5, 7, 4), 16)])
def test_real_path_matches_oracle(ctx, H, sf, sg, m):
    """hd_conv_real (two half-problems packed as one complex problem) equals the
    real part of the oracle's convolution of the same real data."""
    torch_ = pytest.importorskip("torch")
    rng = np.random.default_rng(800 + len(sf) + sf[0])
    f = rng.uniform(-1, 1, sf)
    g = rng.uniform(-1, 1, sg)
    plan = H.Plan.make(len(sf), [{"m": m, "C": 1, "S": 2}] * len(sf))
    h = ctx.conv_real(torch_.from_numpy(f).cuda(), torch_.from_numpy(g).cuda(), plan=plan).cpu().numpy()
    ref = oracle.conv(f.astype(complex), g.astype(complex))
    assert np.abs(ref.imag).max() < 1e-9
    assert h.shape == ref.shape and oracle.rel_l2(h, ref.real) < 1e-11


@pytest.mark.parametrize("sf,sg", [((300, 4000), (20, 300)),    # x: q = 9 -> pack / unpack fused
                                   ((301, 4000), (31, 300)),    # odd rows: the last pair has no im row
                                   ((40, 4096), (255, 255)),    # g taller than f's half: A < L_g
                                   ((7, 4600), (2, 9))])        # x: p_f = 9 > 8 -> unfused fallback
def test_real_path_fused_x_passes(ctx, H, sf, sg):
    """hd_conv_real with the real-pair input / real-split output modes of the staged
    q = 9 x passes (and the fix-up of the rows where two halves overlap)."""
    torch_ = pytest.importorskip("torch")
    rng = np.random.default_rng(820 + sf[0])
    f = rng.uniform(-1, 1, sf)
    g = rng.uniform(-1, 1, sg)
    h = ctx.conv_real(torch_.from_numpy(f).cuda(), torch_.from_numpy(g).cuda()).cpu().numpy()
    ref = oracle.conv(f.astype(complex), g.astype(complex)).real
    assert h.shape == ref.shape and oracle.rel_l2(h, ref) < 1e-11


def test_real_path_batched_and_c64(ctx, H):
    torch_ = pytest.importorskip("torch")
    rng = np.random.default_rng(811)
    f = rng.uniform(-1, 1, (3, 77, 50))
    g = rng.uniform(-1, 1, (3, 9, 12))
    h = ctx.conv_real(torch_.from_numpy(f).cuda(), torch_.from_numpy(g).cuda(), batch=True).cpu().numpy()
    for b in range(3):
        assert oracle.rel_l2(h[b], oracle.conv(f[b].astype(complex), g[b].astype(complex)).real) < 1e-11
    f32, g32 = f[0].astype(np.float32), g[0].astype(np.float32)
    h32 = ctx.conv_real(torch_.from_numpy(f32).cuda(), torch_.from_numpy(g32).cuda()).cpu().numpy()
    assert oracle.rel_l2(h32, oracle.conv(f32.astype(complex), g32.astype(complex)).real) < 1e-5


def test_alias_2d(ctx, H):
    f, g = synth.random_pair(71, (10, 12), (7, 5))
    p = H.Plan.make(2, [{"m": 4}, {"m": 4}], flags=H.HD_FLAG_ALLOW_ALIAS)
    h = host(ctx.conv(dev(f), dev(g), M=[12, 8], plan=p))
    want = oracle.alias_fold(oracle.conv(f, g), [12, 8])
    assert h.shape == want.shape and oracle.rel_l2(h, want) < 1e-11


def test_tune_small(ctx, H):
    p = ctx.tune(H.HD_C128, [200, 300], [31, 17], reps=2)
    log = ctx.hd_tune_log()
    assert len(log) >= 2 and p.tuned_seconds > 0
    assert abs(p.tuned_seconds - min(t for _, t in log)) <= 1e-9 * p.tuned_seconds
    f, g = synth.random_pair(80, (200, 300), (31, 17))
    h = host(ctx.conv(dev(f), dev(g), plan=p))
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11


# ---------------------------------------------------------------- staged warp engine (m = 512)
# hd_s512.cuh runs every m = 512 complex-double pass with one line per CTA (C = 1)
# and an automatic engine choice; HD_FLAG_GENERIC_FFT forces the generic engine.
@pytest.mark.parametrize("shape,S", [(((600, 700), (100, 90)), 2), (((1000, 513), (255, 300)), 2),
                                     (((1000, 513), (255, 300)), 1), (((700, 1200), (33, 511)), 4),
                                     (((513, 2100), (512, 77)), 16)])
def test_s512_engine_matches_oracle_and_generic(ctx, H, shape, S):
    (sf, sg) = shape
    f, g = synth.random_pair(90, sf, sg)
    ref = oracle.conv(f, g)
    axes = [{"m": 512, "C": 1, "S": S}, {"m": 512, "C": 1, "S": S}]
    hw = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(2, axes)))
    hg = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(2, axes, flags=H.HD_FLAG_GENERIC_FFT)))
    assert oracle.rel_l2(hw, ref) < 1e-11
    assert oracle.rel_l2(hg, ref) < 1e-11


@pytest.mark.parametrize("shape", [
    ((1, 1), (1, 1)),            # single element: q = 1, p = 1, one output
    ((300, 200), (100, 100)),    # q = 1 on both axes
    ((17, 3), (512, 2)),         # short input of exactly m = 512 rows (p_g = 1, not pruned)
    ((600, 513), (257, 40)),     # L_g = 257 (just past the pruned half), x: p = 2 from 513
    ((1100, 90), (40, 5000)),    # x: the long input is g (swapped roles), q = 10
    ((2, 5000), (1, 600)),       # x: q = 11 (largest staged q), p_f = 10 > 8 -> generic fwd
])
def test_s512_engine_edge_cases(ctx, H, shape):
    """Degenerate and boundary shapes through the staged m = 512 plans (automatic
    engine choice falls back to the generic engine where the staged one does not
    apply; both must agree with the oracle)."""
    sf, sg = shape
    f, g = synth.random_pair(840 + sf[0], sf, sg)
    axes = [{"m": 512, "C": 1, "S": 2}, {"m": 512, "C": 1, "S": 2}]
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(2, axes)))
    ref = oracle.conv(f, g)
    assert h.shape == ref.shape and oracle.rel_l2(h, ref) < 1e-11


@pytest.mark.parametrize("shape", [((3000, 2500), (500, 300)), ((4000, 1700), (230, 4000))])
def test_s512_engine_large_q_sampled(ctx, H, shape):
    """q up to 12 along x (fwd/inv passes) and q = 7..9 along the convolution axis,
    ragged last blocks; checked on a seeded sample of outputs with the direct sum."""
    (sf, sg) = shape
    f, g = synth.random_pair(91, sf, sg)
    axes = [{"m": 512, "C": 1, "S": 2}, {"m": 512, "C": 1, "S": 2}]
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(2, axes)))
    idx = synth.sample_indices(h.shape, n_random=1500)
    ref = oracle.conv_sampled(f, g, idx)
    assert oracle.rel_l2(h[tuple(idx.T)], ref) < 1e-11


def test_s512_engine_batched_2d(ctx, H):
    f = np.stack([synth.random_pair(92 + b, (300, 700), (40, 50))[0] for b in range(3)])
    g = np.stack([synth.random_pair(95 + b, (300, 700), (40, 50))[1] for b in range(3)])
    axes = [{"m": 512, "C": 1, "S": 2}, {"m": 512, "C": 1, "S": 2}]
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(2, axes), batch=True))
    for b in range(3):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11


@pytest.mark.parametrize("N,sf,sg", [(3, (1200, 300), (700, 40)), (1, (900, 200), (600, 70)),
                                     (6, (700, 130), (520, 20)), (2, (2048, 90), (1000, 33))])
def test_s512_multipair_conv(ctx, H, N, sf, sg):
    """Staged multi-pair convolution pass (MODE_MCONV: h = sum_k f_k * g_k, short
    inputs of several blocks, q <= 6 along the convolution axis)."""
    fs, gs = [], []
    for k in range(N):
        f, g = synth.random_pair(730 + 10 * N + k, sf, sg)
        fs.append(f); gs.append(g)
    axes = [{"m": 512, "C": 1, "S": 2}, {"m": 512, "C": 1, "S": 2}]
    h = host(ctx.multiconv([dev(f) for f in fs], [dev(g) for g in gs], plan=H.Plan.make(2, axes)))
    assert oracle.rel_l2(h, oracle.multiconv(fs, gs)) < 1e-11


@pytest.mark.parametrize("L,q", [(512, 1), (1000, 2), (4000, 8), (4096, 9)])
def test_s512_residues_match_dft(ctx, H, L, q):
    x = synth.random_pair(L, (3, L), (1,))[0]
    X = host(ctx.hd_forward_residues(dev(x), 512, q))
    perm = H.hd_spectral_permutation(512)
    full = [oracle.dft(x[l], q * 512, +1) for l in range(3)]
    for l in range(3):
        for r in range(q):
            got = np.empty(512, complex)
            got[perm] = X[l, r * 512:(r + 1) * 512]
            assert oracle.rel_l2(got, full[l][r::q]) < 1e-12


# ---------------------------------------------------------------- staged engine (m = 128, complex64)
# hd_s128.cuh runs every pass of a complex64 axis with m = 128, C = 4 lines per item
# and D = q <= 8 (automatic engine choice); HD_ENGINE_S128 counts its launches.
S128_AXES = [{"m": 128, "C": 4, "S": 4}] * 3


@pytest.mark.parametrize("sf,sg,S", [
    ((9, 130, 260), (4, 10, 9), 4),      # q = 1, 2, 3; plain rows by bulk copies, p_f = 3 along x
    ((40, 33, 129), (100, 7, 129), 4),   # odd rows (per-thread loads), 33 lines (ragged group)
    ((3, 5, 900), (2, 3, 120), 4),       # x: q = 8, p_f = 8 (largest staged q / p)
    ((30, 64, 200), (9, 64, 57), 8),     # tiles of 8 lines: a 4-line group is half a tile
    ((30, 64, 200), (9, 64, 57), 2),     # tiles of 2 lines: no tensor boxes (per-thread copies)
    ((300, 4, 4), (250, 2, 3), 4),       # q = 5 (compile-time-q kernel) along z, p_f = 3, p_g = 2
    ((4, 300, 6), (2, 250, 3), 4),       # ... along y
    ((4, 6, 512), (2, 3, 129), 4),       # ... along x: the config-4 row lengths (p_f = 4, p_g = 2)
])
def test_s128_engine_3d(ctx, H, sf, sg, S):
    f, g = synth.random_pair(1280 + sf[2] + S, sf, sg, dtype=np.complex64)
    ref = oracle.conv(f, g)
    axes = [{"m": 128, "C": 4, "S": S}] * 3
    n0 = ctx.engine_launches(H.HD_ENGINE_S128)
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(3, axes)))
    assert ctx.engine_launches(H.HD_ENGINE_S128) - n0 == 7
    hg = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(3, axes, flags=H.HD_FLAG_GENERIC_FFT)))
    assert oracle.rel_l2(h, ref) < 1e-5
    assert oracle.rel_l2(hg, ref) < 1e-5


def test_s128_engine_batched_multipair_window(ctx, H):
    """Batched 3-D, N = 2 pairs (forward passes with two arrays; the convolution pass
    of several pairs runs on the generic engine), and an output window (plain stores)."""
    fs, gs = zip(*[synth.random_pair(1300 + k, (12, 40, 150), (5, 9, 20), dtype=np.complex64)
                   for k in range(2)])
    h = host(ctx.multiconv([dev(x) for x in fs], [dev(x) for x in gs], plan=H.Plan.make(3, S128_AXES)))
    assert oracle.rel_l2(h, oracle.multiconv(list(fs), list(gs))) < 1e-5
    f = np.stack([synth.random_pair(1310 + b, (10, 20, 300), (3, 6, 30), dtype=np.complex64)[0] for b in range(3)])
    g = np.stack([synth.random_pair(1320 + b, (10, 20, 300), (3, 6, 30), dtype=np.complex64)[1] for b in range(3)])
    n0 = ctx.engine_launches(H.HD_ENGINE_S128)
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(3, S128_AXES), batch=True))
    assert ctx.engine_launches(H.HD_ENGINE_S128) - n0 == 7
    for b in range(3):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-5
    lo, n = [1, 3, 17], [10, 20, 250]
    h = host(ctx.conv_window([dev(f[0])], [dev(g[0])], lo, n, plan=H.Plan.make(3, S128_AXES)))
    ref = oracle.conv(f[0], g[0])[1:11, 3:23, 17:267]
    assert oracle.rel_l2(h, ref) < 1e-5


# ---------------------------------------------------------------- row f1: Lambda > 1 (1-D)
@pytest.mark.parametrize("Lf,Lg,m,Lam,dtype", [
    (7, 30, 4, 2, np.complex128), (13, 50, 4, 4, np.complex128), (100, 1000, 32, 4, np.complex128),
    (255, 4096, 256, 2, np.complex128), (1, 9, 2, 2, np.complex128), (64, 64, 16, 1, np.complex128),
    (300, 5000, 64, 8, np.complex64), (129, 512, 64, 2, np.complex64)])
def test_lambda_conv_matches_oracle(ctx, H, Lf, Lg, m, Lam, dtype):
    f, g = synth.random_pair(1400 + Lf, (3, Lf), (3, Lg), dtype=dtype)
    h = host(ctx.conv1d_lambda(dev(f), dev(g), m, Lam))
    for b in range(3):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < TOL[dtype]
    if Lg <= 200:  # the step-by-step oracle of the construction itself (slow)
        assert oracle.rel_l2(h[0], oracle.lambda_conv(f[0], g[0], m, Lam)) < TOL[dtype]


def test_lambda_conv_config2_shape_and_padding(ctx, H):
    """The config-2 pair (3000 (*) 8192, batch 8 here) with Lambda = 4, m = 256, and an
    explicit M above L_out; sampled lines against the direct sum."""
    f, g = synth.random_pair(1450, (8, 3000), (8, 8192))
    h = host(ctx.conv1d_lambda(dev(f), dev(g), 256, 4))
    h2 = host(ctx.conv1d_lambda(dev(f), dev(g), 256, 4, M=12288))
    for b in (0, 7):
        ref = oracle.conv(f[b], g[b])
        assert oracle.rel_l2(h[b], ref) < 1e-11 and oracle.rel_l2(h2[b], ref) < 1e-11
    with pytest.raises(H.HDError):
        ctx.conv1d_lambda(dev(g), dev(f), 256, 4)  # L_f > L_g
    with pytest.raises(H.HDError):
        ctx.conv1d_lambda(dev(f), dev(g), 256, 4, M=100)


# ---------------------------------------------------------------- 1-D long lines: two-CTA clusters
# hd_s512c.cuh: m = 512, 12 <= q <= 22, residues split over a cluster of two CTAs,
# partial unfolds exchanged through distributed shared memory.
@pytest.mark.parametrize("B,Lf,Lg,m", [(4, 8192, 3000, 512),   # config 2's pair: q = 22
                                        (3, 6000, 200, 512),    # q = 13 (odd: 7 / 6 residues)
                                        (2, 6000, 145, 512),    # L_out = 12 x 512 exactly: q = 12
                                        (5, 300, 9000, 512),    # the long input is g
                                        (1, 5000, 4000, 512),   # p_f = 10, p_g = 8
                                        (4, 8192, 3000, 2048),  # m = 2048 (four warps per residue): q = 6
                                        (3, 9000, 500, 2048),   # q = 5 (3 / 2 residues)
                                        (2, 6000, 200, 2048),   # q = 4 (1 / 3 residues)
                                        (2, 300, 11000, 2048)]) # swapped roles, p_g = 6
def test_s512c_cluster_conv1d(ctx, H, B, Lf, Lg, m):
    f, g = synth.random_pair(1500 + Lf + m, (B, Lf), (B, Lg))
    plan = H.Plan.make(1, [{"m": m, "C": 1}])
    # m = 2048 runs on the one-CTA-per-line engine (hd_s2048r.cuh), which superseded
    # the two-CTA cluster variant at that size
    eng = H.HD_ENGINE_S512C if m == 512 else H.HD_ENGINE_S2048R
    n0 = ctx.engine_launches(eng)
    h = host(ctx.conv(dev(f), dev(g), plan=plan, batch=True))
    assert ctx.engine_launches(eng) - n0 == 1
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11


def test_s512c_shared_g_and_window(ctx, H):
    f = np.stack([synth.random_pair(1520 + b, (7000,), (1,))[0] for b in range(3)])
    g = synth.random_pair(1530, (1,), (2500,))[1]
    plan = H.Plan.make(1, [{"m": 512, "C": 1}])
    h = host(ctx.conv(dev(f), dev(g), plan=plan, batch=True, shared_g=True))
    for b in range(3):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g)) < 1e-11
    lo, n = [1234], [5000]
    hw = host(ctx.conv_window([dev(f[0])], [dev(g)], lo, n, plan=plan))
    assert oracle.rel_l2(hw, oracle.conv(f[0], g)[1234:6234]) < 1e-11


@pytest.mark.parametrize("sf,sg", [((300, 500), (40, 90)),     # x: q = 5 (compile-time kernels), y: q = 3
                                   ((129, 640), (3, 1)),       # x: L_out = 640 exactly
                                   ((1000, 77), (25, 51))])    # y: q = 9 (runtime-q kernel, 288 threads)
def test_s128_engine_2d(ctx, H, sf, sg):
    """The staged complex-float engine on both axes of a 2-D problem."""
    f, g = synth.random_pair(1600 + sf[0], sf, sg, dtype=np.complex64)
    plan = H.Plan.make(2, [{"m": 128, "C": 4, "S": 4}] * 2)
    n0 = ctx.engine_launches(H.HD_ENGINE_S128)
    h = host(ctx.conv(dev(f), dev(g), plan=plan))
    assert ctx.engine_launches(H.HD_ENGINE_S128) - n0 >= 3
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-5


# ---------------------------------------------------------------- HD_FLAG_GRAPH (CUDA-graph replay)
@pytest.mark.parametrize("sf,sg,axes", [((64,), (40,), [{"m": 32}]),
                                        ((300, 700), (40, 50), [{"m": 512, "C": 1, "S": 2}] * 2),
                                        ((20, 30, 40), (5, 6, 7), [{"m": 16, "C": 2, "S": 2}] * 3)])
def test_graph_replay_matches_and_tracks_inputs(ctx, H, sf, sg, axes):
    """The second identical call replays the graph captured on the first; the graph
    reads the buffers at replay time (new contents, same pointers -> new result)."""
    f, g = synth.random_pair(1700 + len(sf), sf, sg)
    plan = H.Plan.make(len(sf), axes, flags=H.HD_FLAG_GRAPH)
    fd, gd = dev(f), dev(g)
    h = ctx.conv(fd, gd, plan=plan)
    r0 = ctx.graph_replays()
    ctx.conv(fd, gd, plan=plan, h=h)
    assert ctx.graph_replays() == r0 + 1
    assert oracle.rel_l2(host(h), oracle.conv(f, g)) < 1e-11
    f2, g2 = synth.random_pair(1710 + len(sf), sf, sg)
    fd.copy_(torch.from_numpy(f2).cuda())
    gd.copy_(torch.from_numpy(g2).cuda())
    ctx.conv(fd, gd, plan=plan, h=h)
    assert ctx.graph_replays() == r0 + 2
    assert oracle.rel_l2(host(h), oracle.conv(f2, g2)) < 1e-11


def test_graph_dropped_when_workspace_grows(H):
    """A larger problem reallocates the context workspace: the captured graphs (which
    address the old workspace) are dropped and the next identical call re-captures."""
    c = H.Context(0)
    try:
        f, g = synth.random_pair(1720, (40, 50), (9, 7))
        plan = H.Plan.make(2, [{"m": 32, "C": 2, "S": 2}] * 2, flags=H.HD_FLAG_GRAPH)
        fd, gd = dev(f), dev(g)
        h = c.conv(fd, gd, plan=plan)
        c.conv(fd, gd, plan=plan, h=h)
        assert c.graph_replays() == 1
        F, G = synth.random_pair(1721, (600, 700), (50, 40))
        c.conv(dev(F), dev(G))                      # grows the workspace
        c.conv(fd, gd, plan=plan, h=h)              # re-captured, not replayed
        assert c.graph_replays() == 1
        c.conv(fd, gd, plan=plan, h=h)
        assert c.graph_replays() == 2
        assert oracle.rel_l2(host(h), oracle.conv(f, g)) < 1e-11
    finally:
        c.close()


@pytest.mark.parametrize("sf,sg", [((40, 4000), (9, 300)),      # x: q = 9 -> f and g rows in one launch
                                   ((3, 4096), (255, 255)),     # more g rows than f rows
                                   ((257, 4096), (1, 255))])    # one g row
def test_merged_forward_launch(ctx, H, sf, sg):
    """2-D, one pair, x on the staged q = 9 kernel: the f rows and the g rows go
    through one forward launch (PassArgs fam2); three launches per convolution."""
    f, g = synth.random_pair(1800 + sf[0], sf, sg)
    plan = H.Plan.make(2, [{"m": 512, "C": 1, "S": 2}] * 2)
    n0 = ctx.launch_count()
    h = host(ctx.conv(dev(f), dev(g), plan=plan))
    assert ctx.launch_count() - n0 == 3
    idx = synth.sample_indices(h.shape, n_random=400)
    assert oracle.rel_l2(h[tuple(idx.T)], oracle.conv_sampled(f, g, idx)) < 1e-11


@pytest.mark.parametrize("dtype,m,C,L,q", [(np.complex128, 512, 1, 3000, 7),
                                           (np.complex64, 128, 4, 500, 5),
                                           (np.complex128, 512, 1, 4096, 9)])
def test_pass_staged_order_round_trip(ctx, H, dtype, m, C, L, q):
    """hd_pass with HD_FLAG_STAGED_ORDER: forward then inverse on the staged engine in
    its own spectral order returns q m x exactly as the documented-order passes do;
    the flag is refused (HD_ERR_UNSUPPORTED) where no staged engine applies."""
    nl = 8
    x = synth.random_pair(1900 + m, (nl, L), (1,))[0].astype(dtype)
    dt = H.HD_C128 if dtype == np.complex128 else H.HD_C64
    M1 = q * m
    xd = dev(x)
    X = torch.empty(nl * M1, dtype=xd.dtype, device="cuda")
    y = torch.empty(nl * L, dtype=xd.dtype, device="cuda")

    def desc(mode, inp, Lin, s_in, out, Lout, s_out):
        d = H.PassDesc()
        d.mode, d.npairs, d.nlines, d.nbatch, d.M = mode, 1, nl, 1, M1
        d.axis.m, d.axis.C, d.axis.D, d.axis.threads = m, C, 0, 0
        d.in_f = H.Lines.make([inp.data_ptr()], Lin, s_l=s_in)
        d.out = H.Lines.make([out.data_ptr()], Lout, s_l=s_out)
        d.flags = H.HD_FLAG_STAGED_ORDER
        return d
    n0 = ctx.engine_launches(H.HD_ENGINE_S512) + ctx.engine_launches(H.HD_ENGINE_S128)
    ctx.hd_pass(dt, desc(H.HD_PASS_FWD, xd, L, L, X, M1, M1))
    ctx.hd_pass(dt, desc(H.HD_PASS_INV, X, M1, M1, y, L, L))
    assert ctx.engine_launches(H.HD_ENGINE_S512) + ctx.engine_launches(H.HD_ENGINE_S128) - n0 == 2
    got = host(y).reshape(nl, L) / M1
    assert oracle.rel_l2(got, x) < (1e-13 if dtype == np.complex128 else 1e-5)
    bad = desc(H.HD_PASS_FWD, xd, L, L, X, M1, M1)
    bad.axis.C = 2 if C == 1 else 1   # no staged engine with this line count
    with pytest.raises(H.HDError):
        ctx.hd_pass(dt, bad)


# ---------------------------------------------------------------- threads
def test_contexts_on_concurrent_threads(H):
    """Two host threads, each with its own context and stream, convolve different
    problems at once (staged and generic engines, > 48 KB of shared memory): the
    launchers' per-device caches are shared and locked (hd_kernels.cu)."""
    import threading
    cases = [(((1100, 700), (255, 60)), np.complex128), (((300, 260), (31, 17)), np.complex128),
             (((150, 18, 24), (5, 7, 4)), np.complex64), (((5000,), (900,)), np.complex128)]
    data = [synth.random_pair(900 + i, Lf, Lg, dtype=dt) for i, ((Lf, Lg), dt) in enumerate(cases)]
    results, errors = {}, []

    def worker(k):
        try:
            c = H.Context(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    for i in range(k, len(cases), 2):
                        f, g = data[i]
                        h = c.conv(dev(f), dev(g), stream=s)
                        s.synchronize()
                        results[(i, rep)] = h.cpu().numpy()
            c.close()
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errors, errors
    for (i, rep), h in results.items():
        f, g = data[i]
        tol = 1e-11 if cases[i][1] == np.complex128 else 1e-5
        assert oracle.rel_l2(h, oracle.conv(f, g)) < tol, (i, rep)
    assert len(results) == 3 * len(cases)


# ---------------------------------------------------------------- context scratch
def test_graph_survives_lambda_workspace_growth(H):
    """A larger hd_conv1d_lambda regrows the context workspace: captured graphs that
    addressed the old one are dropped (re-captured), never replayed on freed memory."""
    c = H.Context(0)
    try:
        f, g = synth.random_pair(1730, (40, 50), (9, 7))
        plan = H.Plan.make(2, [{"m": 32, "C": 2, "S": 2}] * 2, flags=H.HD_FLAG_GRAPH)
        fd, gd = dev(f), dev(g)
        h = c.conv(fd, gd, plan=plan)
        c.conv(fd, gd, plan=plan, h=h)
        assert c.graph_replays() == 1
        a, b = synth.random_pair(1731, (64, 3000), (64, 8192))
        hl = host(c.conv1d_lambda(dev(a), dev(b), m=512, Lambda=2))   # grows ctx->ws
        assert oracle.rel_l2(hl[5], oracle.conv(a[5], b[5])) < 1e-11
        c.conv(fd, gd, plan=plan, h=h)               # re-captured, not replayed
        assert c.graph_replays() == 1
        c.conv(fd, gd, plan=plan, h=h)
        assert c.graph_replays() == 2
        assert oracle.rel_l2(host(h), oracle.conv(f, g)) < 1e-11
    finally:
        c.close()


def test_shared_scratch_ordered_across_streams(H):
    """Calls without a caller workspace share the context scratch: calls enqueued
    back to back on two different streams (no host sync between) must not overwrite
    each other's intermediates."""
    c = H.Context(0)
    try:
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        cases = [synth.random_pair(1740 + i, (700, 900), (120, 77)) for i in range(4)]
        ins = [(dev(f), dev(g)) for f, g in cases]
        torch.cuda.synchronize()
        outs = []
        for i, (fd, gd) in enumerate(ins):
            s = s1 if i % 2 == 0 else s2
            with torch.cuda.stream(s):
                outs.append(c.conv(fd, gd, stream=s))
        rf, rg = synth.random_pair(1745, (300, 200), (31, 17))
        with torch.cuda.stream(s2):
            rr = c.conv_real(dev(rf.real.copy()), dev(rg.real.copy()), stream=s2)
        torch.cuda.synchronize()
        for (f, g), h in zip(cases, outs):
            idx = synth.sample_indices(h.shape, n_random=300)
            got = h.cpu().numpy()[tuple(idx.T)]
            assert oracle.rel_l2(got, oracle.conv_sampled(f, g, idx)) < 1e-11
        assert oracle.rel_l2(rr.cpu().numpy(), oracle.conv(rf.real, rg.real)) < 1e-11
    finally:
        c.close()


def test_binding_validates_operands(ctx, H):
    """The binding refuses operands the kernels would misread."""
    f, g = synth.random_pair(1750, (50,), (20,))
    fd, gd = dev(f), dev(g)
    with pytest.raises(TypeError):
        ctx.conv(fd, gd.to(torch.complex64))
    with pytest.raises(ValueError):
        ctx.conv(fd[::2], gd)
    with pytest.raises(ValueError):
        ctx.conv(fd.unsqueeze(0).expand(4, 50).contiguous(), gd.unsqueeze(0).expand(3, 20).contiguous(), batch=True)
    with pytest.raises(ValueError):
        ctx.conv(fd, gd, h=torch.empty(10, dtype=fd.dtype, device="cuda"))
    with pytest.raises(ValueError):
        ctx.multiconv([fd, fd], [gd, gd[:10].contiguous()])
    with pytest.raises(ValueError):
        ctx.hd_conv_host([f], [g], np.zeros(10, dtype=np.complex128), ndim=1)
    with pytest.raises(ValueError):
        ctx.conv(fd.cpu(), gd.cpu())


def test_shared_g_does_not_mutate_plan(ctx, H):
    """conv(..., shared_g=True, plan=p) must not set HD_FLAG_SHARED_G on p: a later
    per-entry-g call with the same plan uses every g_b."""
    B = 3
    f, _ = synth.random_pair(1760, (B, 200), (1,))
    g = synth.random_pair(1761, (B, 60), (1,))[0]
    plan = H.Plan.make(1, [{"m": 64}])
    ctx.conv(dev(f), dev(g[0]), batch=True, shared_g=True, plan=plan)
    assert not (plan.flags & H.HD_FLAG_SHARED_G)
    h = host(ctx.conv(dev(f), dev(g), batch=True, plan=plan))
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11



# ---------------------------------------------------------------- image filter (row f3)
@pytest.mark.parametrize("kid", range(8))
@pytest.mark.parametrize("channel_last,dtype", [(True, np.float64), (False, np.float64), (True, np.float32)])
def test_filter_image_dictionary(ctx, H, kid, channel_last, dtype):
    """The paper's image-filter demo on a synthetic 3-channel
    100 x 120 image of integer pixel values: every channel convolved with dictionary
    kernel `kid`, real part kept, a window of the full result, against the oracle."""
    s = synth.Stream(4000 + kid)
    img = np.floor(s.real_uniform((100, 120, 3), 0.0, 256.0))
    name, w = H.filter_kernel(kid)
    n = w.shape[0]
    lo, nn = [1, 2], [100 + n - 3, 120 + n - 4]
    x = img if channel_last else np.ascontiguousarray(np.transpose(img, (2, 0, 1)))
    out = host(ctx.filter_image(dev(x.astype(dtype)), kid, window=(lo, nn), channel_last=channel_last))
    tol = 1e-11 if dtype == np.float64 else 1e-5
    for c in range(3):
        ref = np.real(oracle.conv(img[:, :, c], w))[lo[0]:lo[0] + nn[0], lo[1]:lo[1] + nn[1]]
        got = out[:, :, c] if channel_last else out[c]
        assert oracle.rel_l2(got, ref) < tol, (name, c)


def test_explicit_variant_tuned_plan(ctx, H):
    """hd_tune_explicit tunes the padded problem's own plan; hd_conv_explicit(plan=None)
    then uses it, and an HD_FLAG_EXPLICIT_PLAN plan is honoured as the padded plan."""
    f, g = synth.random_pair(4100, (300, 260), (31, 17))
    p = ctx.tune_explicit(H.HD_C128, [300, 260], [31, 17], reps=1)
    assert p.flags & H.HD_FLAG_EXPLICIT_PLAN and p.tuned_seconds > 0
    assert len(ctx.hd_tune_log()) > 10
    h = host(ctx.hd_conv_explicit([dev(f)], [dev(g)]))
    ref = oracle.conv(f, g)
    assert oracle.rel_l2(h, ref) < 1e-11
    own = H.Plan.make(2, [{"m": 64, "C": 2, "S": 4}, {"m": 128, "C": 1, "S": 2}], flags=H.HD_FLAG_EXPLICIT_PLAN)
    h2 = host(ctx.hd_conv_explicit([dev(f)], [dev(g)], plan=own))
    assert oracle.rel_l2(h2, ref) < 1e-11


# ---------------------------------------------------------------- 1-D m = 2048 engine (hd_s2048r.cuh)
@pytest.mark.parametrize("B,Lf,Lg", [(5, 8192, 3000),    # config 2's lines: q = 6, p_f = 4, p_g = 2
                                     (3, 6000, 3000),    # q = 5 (last pair has one residue)
                                     (2, 8192, 8192),    # q = 8, p = 4 both
                                     (4, 1000, 9000),    # f shorter than g (roles as given)
                                     (3, 2048, 1),       # q = 1
                                     (7, 4097, 2049)])   # ragged blocks
def test_s2048r_engine(ctx, H, B, Lf, Lg):
    f, g = synth.random_pair(4200 + Lf + Lg, (B, Lf), (B, Lg))
    plan = H.Plan.make(1, [{"m": 2048}])
    n0 = ctx.engine_launches(H.HD_ENGINE_S2048R)
    h = host(ctx.conv(dev(f), dev(g), plan=plan, batch=True))
    assert ctx.engine_launches(H.HD_ENGINE_S2048R) - n0 == 1
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11, b


def test_s2048r_shared_g(ctx, H):
    B = 6
    f, _ = synth.random_pair(4300, (B, 8192), (1,))
    g = synth.random_pair(4301, (3000,), (1,))[0]
    n0 = ctx.engine_launches(H.HD_ENGINE_S2048R)
    h = host(ctx.conv(dev(f), dev(g), plan=H.Plan.make(1, [{"m": 2048}]), batch=True, shared_g=True))
    assert ctx.engine_launches(H.HD_ENGINE_S2048R) - n0 == 1
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g)) < 1e-11


# ---------------------------------------------------------------- 1-D m = 4096 engine (hd_s4096r.cuh)
@pytest.mark.parametrize("B,Lf,Lg", [(5, 8192, 3000),    # config 2's lines: q = 3, p_f = 2, p_g = 1
                                     (3, 5000, 200),     # q = 2
                                     (2, 9000, 5000),    # q = 4, p_f = 3, p_g = 2
                                     (2, 16384, 1),      # q = 4, p_f = 4, L_out = 4 m exactly
                                     (4, 1000, 9000),    # f shorter than g (roles as given)
                                     (3, 4096, 1),       # q = 1 (no residue slots)
                                     (7, 4097, 4097),    # ragged blocks, q = 3
                                     (150, 700, 4000)])  # more lines than SMs on small GPUs' grids
def test_s4096r_engine(ctx, H, B, Lf, Lg):
    f, g = synth.random_pair(4400 + Lf + Lg, (B, Lf), (B, Lg))
    plan = H.Plan.make(1, [{"m": 4096}])
    n0 = ctx.engine_launches(H.HD_ENGINE_S4096R)
    h = host(ctx.conv(dev(f), dev(g), plan=plan, batch=True))
    assert ctx.engine_launches(H.HD_ENGINE_S4096R) - n0 == 1
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11, b


def test_s4096r_shared_g_and_default_plan(ctx, H):
    B = 6
    f, _ = synth.random_pair(4500, (B, 8192), (1,))
    g = synth.random_pair(4501, (3000,), (1,))[0]
    pc = H.hd_plan_complete(H.HD_C128, [8192], [3000], ctx.default_plan(H.HD_C128, [8192], [3000]))
    assert (pc.axis[0].m, pc.axis[0].q, pc.axis[0].D) == (4096, 3, 3), pc.as_dict()
    n0 = ctx.engine_launches(H.HD_ENGINE_S4096R)
    h = host(ctx.conv(dev(f), dev(g), batch=True, shared_g=True))   # default plan: m = 4096, D = q
    assert ctx.engine_launches(H.HD_ENGINE_S4096R) - n0 == 1
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g)) < 1e-11


@pytest.mark.parametrize("m,lo,n", [(4096, 0, 11191),      # the whole output through the window path
                                    (4096, 5, 300),        # inside the first block
                                    (4096, 4000, 5000),    # across blocks 0-2
                                    (4096, 11000, 191),    # the tail
                                    (2048, 3000, 6000)])   # m = 2048: the generic fallback (D lowered)
def test_long_line_windows(ctx, H, m, lo, n):
    """1-D output windows of config 2's line shape on the one-CTA-per-line engine (m = 4096)
    and through the generic fallback of an m = 2048 plan."""
    B, Lf, Lg = 3, 8192, 3000
    f, g = synth.random_pair(4600 + lo, (B, Lf), (B, Lg))
    eng = H.HD_ENGINE_S4096R if m == 4096 else H.HD_ENGINE_GENERIC
    n0 = ctx.engine_launches(eng)
    h = host(ctx.conv_window([dev(f)], [dev(g)], [lo], [n], batch=True, plan=H.Plan.make(1, [{"m": m}])))
    assert ctx.engine_launches(eng) - n0 == 1
    for b in range(B):
        ref = oracle.conv(f[b], g[b])[lo:lo + n]
        assert h[b].shape == ref.shape and oracle.rel_l2(h[b], ref) < 1e-11, b



def test_s4096r_graph_replay(ctx, H):
    """HD_FLAG_GRAPH on the m = 4096 1-D engine (its residue slots live in the context
    workspace): the replay matches the oracle and reads new inputs."""
    B, Lf, Lg = 4, 8192, 3000
    f, g = synth.random_pair(4700, (B, Lf), (B, Lg))
    plan = H.Plan.make(1, [{"m": 4096}], flags=H.HD_FLAG_GRAPH)
    fd, gd = dev(f), dev(g)
    h = ctx.conv(fd, gd, plan=plan, batch=True)
    r0 = ctx.graph_replays()
    f2, g2 = synth.random_pair(4701, (B, Lf), (B, Lg))
    fd.copy_(torch.from_numpy(f2).cuda())
    gd.copy_(torch.from_numpy(g2).cuda())
    ctx.conv(fd, gd, plan=plan, h=h, batch=True)
    assert ctx.graph_replays() == r0 + 1
    hh = host(h)
    for b in range(B):
        assert oracle.rel_l2(hh[b], oracle.conv(f2[b], g2[b])) < 1e-11, b
