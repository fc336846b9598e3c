"""Full-size parity at BASELINE.json's configs, in the plan bench.py times
(SURVEY.md §8(d) "Oracle timing": configs 1-3 on ALL outputs; configs 4-5 on
2^16 seeded random output indices plus every corner and the first/last 64
indices along each axis, plus 8 polynomial-identity points).

The oracle is the direct sum of Eq. 4 on the box's host
cores: config 3's full output is ~1.1e12 complex MACs (~1-2 min on 16 cores),
config 2's ~1e11.  The reference for config 3 is computed once per module and
shared by the default-plan, tuned-plan and explicit-variant checks.

Polynomial identity (closed form, involves EVERY output sample): for z uniform
on the unit torus the characters z^o are orthonormal, so E_z |P_e(z)|^2 =
||e||_2^2 for an error e.  A correct result (relL2(h) <= tol) therefore gives
|P_h(z) - sum_k P_fk(z) P_gk(z)| of order tol*||h||_2; the test allows
POLY_C * tol * ||h||_2 (Markov: false-failure probability <= 1/POLY_C^2 per
point) plus the oracle's own Horner rounding bound, (sum_i deg_i + 2) * eps *
(||h||_1 + sum_k ||f_k||_1 ||g_k||_1) for |z_i| = 1.  A corrupted block of k
outputs of typical magnitude |h| moves |P_e| by ~sqrt(k)|h| per point.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = {"c128": 1e-11, "c64": 1e-5}
POLY_C = 50.0
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import hdconv
    return hdconv


@pytest.fixture(scope="module")
def ctx(H):
    c = H.Context(0)
    yield c
    c.close()


def _poly_check(fs, gs, h, tol, npts=8):
    """Polynomial identity at npts seeded points of the unit torus (see module doc)."""
    h = np.asarray(h, dtype=np.complex128)
    z = synth.unit_torus_points(npts, h.ndim, seed=99)
    u = oracle.poly_eps()
    Ph = oracle.poly_eval(h, z)
    deg = sum(h.shape) + 2
    Pfg = np.zeros(npts, dtype=np.complex128)
    rnd = deg * u * np.abs(h).sum() + 4 * EPS * np.abs(Ph)
    for f, g in zip(fs, gs):
        Pf, Pg = oracle.poly_eval(f, z), oracle.poly_eval(g, z)
        Pfg += Pf * Pg
        # Horner rounding of P_f, P_g (long double), their double rounding and the product's
        rnd += (deg * u * np.abs(np.asarray(f)).sum() + 2 * EPS * np.abs(Pf)) * np.abs(Pg) \
            + (deg * u * np.abs(np.asarray(g)).sum() + 2 * EPS * np.abs(Pg)) * np.abs(Pf) \
            + 4 * EPS * np.abs(Pf * Pg)
    bound = POLY_C * tol * np.linalg.norm(h.ravel()) + rnd
    dev = np.abs(Ph - Pfg)
    assert np.all(dev <= bound), (dev, bound)
    return dev, bound


def contract_indices(out_shape, n_random=1 << 16, edge=64, per_edge=16, seed=12345):
    """SURVEY §8(d) sample: every corner; for each axis, each of its first and
    last `edge` indices combined with `per_edge` random positions on the other
    axes; plus n_random uniform random output indices."""
    out_shape = [int(v) for v in out_shape]
    nd = len(out_shape)
    s = synth.Stream(seed)
    rows = [[(out_shape[i] - 1) if (c >> i) & 1 else 0 for i in range(nd)] for c in range(1 << nd)]
    for ax in range(nd):
        n = out_shape[ax]
        for e in sorted(set(range(min(edge, n))) | set(range(max(0, n - edge), n))):
            u = s.uniform(per_edge * nd).reshape(per_edge, nd)
            for k in range(per_edge):
                r = [int(u[k, i] * out_shape[i]) for i in range(nd)]
                r[ax] = e
                rows.append(r)
    u = s.uniform(n_random * nd).reshape(n_random, nd)
    rnd = np.floor(u * np.asarray(out_shape, dtype=np.float64)).astype(np.int64)
    idx = np.concatenate([np.asarray(rows, dtype=np.int64).reshape(-1, nd), rnd])
    return np.unique(idx, axis=0)


def _sampled(fs, gs, h, tol, idx):
    ref = oracle.multiconv_sampled(fs, gs, idx)
    got = h[tuple(idx.T)]
    err = oracle.rel_l2(got, ref)
    assert err < tol, err
    return err


def test_contract_indices_cover_edges_and_corners():
    idx = contract_indices((640, 640, 640), n_random=1000)
    for ax in range(3):
        vals = set(idx[:, ax].tolist())
        assert set(range(64)) <= vals and set(range(576, 640)) <= vals
    for c in range(8):
        corner = [639 if (c >> i) & 1 else 0 for i in range(3)]
        assert (idx == corner).all(axis=1).any()


def test_config1_full(ctx, H):
    d = synth.config_inputs(1)
    f, g = d["f"][0], d["g"][0]
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(),
                 plan=H.Plan.make(1, [{"m": 32}]))
    assert oracle.rel_l2(h.cpu().numpy(), oracle.conv(f, g)) < 1e-11


def test_config2_full(ctx, H):
    """All 4096 rows x 11191 outputs against the direct sum."""
    d = synth.config_inputs(2)
    f, g = d["f"][0], d["g"][0]
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(), batch=True).cpu().numpy()
    assert h.shape == (4096, 11191)
    worst = 0.0
    num = den = 0.0
    for b in range(4096):
        ref = oracle.conv(f[b], g[b])
        e = h[b] - ref
        num += float(np.vdot(e, e).real)
        den += float(np.vdot(ref, ref).real)
        worst = max(worst, oracle.rel_l2(h[b], ref))
    assert np.sqrt(num / den) < 1e-11 and worst < 1e-11, (np.sqrt(num / den), worst)
    _poly_check([f[0]], [g[0]], h[0], 1e-11)


@pytest.fixture(scope="module")
def config3():
    d = synth.config_inputs(3)
    f, g = d["f"][0], d["g"][0]
    return f, g, oracle.conv(f, g)


@pytest.mark.parametrize("tuned", [False, True])
def test_config3_full(ctx, H, config3, tuned):
    """All 4350^2 outputs against the direct sum."""
    f, g, ref = config3
    plan = ctx.tune(H.HD_C128, [4096, 4096], [255, 255], reps=3) if tuned else None
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(), plan=plan).cpu().numpy()
    assert h.shape == (4350, 4350)
    err = oracle.rel_l2(h, ref)
    assert err < 1e-11, err
    rowerr = np.linalg.norm(h - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rowerr.max() < 1e-11, rowerr.max()


def test_config3_explicit_variant(ctx, H, config3):
    f, g, ref = config3
    h = ctx.hd_conv_explicit([torch.from_numpy(f).cuda()], [torch.from_numpy(g).cuda()]).cpu().numpy()
    assert oracle.rel_l2(h, ref) < 1e-11


def test_config4_full(ctx, H):
    d = synth.config_inputs(4)
    f, g = d["f"][0], d["g"][0]
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()).cpu().numpy()
    assert h.shape == (640, 640, 640) and h.dtype == np.complex64
    idx = contract_indices(h.shape)
    assert idx.shape[0] > (1 << 16)
    _sampled([f], [g], h, 1e-5, idx)
    _poly_check([f], [g], h, 1e-5)


def test_config5_full(ctx, H):
    d = synth.config_inputs(5)
    fs, gs = d["f"], d["g"]
    plan = ctx.tune(H.HD_C128, [2048, 2048], [1024, 1536], N=6, reps=2)
    h = ctx.multiconv([torch.from_numpy(a).cuda() for a in fs],
                      [torch.from_numpy(a).cuda() for a in gs], plan=plan).cpu().numpy()
    assert h.shape == (3071, 3583)
    idx = contract_indices(h.shape)
    assert idx.shape[0] > (1 << 16)
    _sampled(fs, gs, h, 1e-11, idx)
    _poly_check(fs, gs, h, 1e-11)
