"""Full-size parity at BASELINE.json's configs, in the plan bench.py times.

The oracle cannot convolve these sizes in seconds, so it checks (a) a seeded
sample of output indices (every corner, the first/last indices along each
axis, random interior points) with the direct sum, and (b) the generating
polynomial identity P_h(z) = P_f(z) P_g(z) on the unit torus, which involves
EVERY output sample: |P_h - P_f P_g| <= tol * sqrt(#out) * ||h||_2 is a
necessary consequence of relL2(h) <= tol."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = {"c128": 1e-11, "c64": 1e-5}


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import hdconv
    return hdconv


@pytest.fixture(scope="module")
def ctx(H):
    c = H.Context(0)
    yield c
    c.close()


def _poly_check(fs, gs, h, tol, npts=3):
    nd = h.ndim
    z = synth.unit_torus_points(npts, nd, seed=99)
    Ph = oracle.poly_eval(h, z)
    Pfg = sum(oracle.poly_eval(f, z) * oracle.poly_eval(g, z) for f, g in zip(fs, gs))
    bound = tol * np.sqrt(h.size) * np.linalg.norm(h.ravel())
    assert np.max(np.abs(Ph - Pfg)) <= bound, (np.max(np.abs(Ph - Pfg)), bound)


def _sampled(fs, gs, h, tol, n_random):
    idx = synth.sample_indices(h.shape, n_random=n_random)
    ref = oracle.multiconv_sampled(fs, gs, idx)
    got = h[tuple(idx.T)]
    err = oracle.rel_l2(got, ref)
    assert err < tol, err
    return err


def test_config1_full(ctx, H):
    d = synth.config_inputs(1)
    f, g = d["f"][0], d["g"][0]
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(),
                 plan=H.Plan.make(1, [{"m": 32}]))
    assert oracle.rel_l2(h.cpu().numpy(), oracle.conv(f, g)) < 1e-11


def test_config2_full(ctx, H):
    d = synth.config_inputs(2)
    f, g = d["f"][0], d["g"][0]
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(), batch=True).cpu().numpy()
    assert h.shape == (4096, 11191)
    rows = np.unique((synth.Stream(5).uniform(12) * 4096).astype(int).tolist() + [0, 4095])
    ref = np.stack([oracle.conv(f[b], g[b]) for b in rows])
    assert oracle.rel_l2(h[rows], ref) < 1e-11
    for b in rows[:3]:
        _poly_check([f[b]], [g[b]], h[b], 1e-11)


@pytest.mark.parametrize("tuned", [False, True])
def test_config3_full(ctx, H, tuned):
    d = synth.config_inputs(3)
    f, g = d["f"][0], d["g"][0]
    plan = ctx.tune(H.HD_C128, [4096, 4096], [255, 255], reps=3) if tuned else None
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(), plan=plan).cpu().numpy()
    assert h.shape == (4350, 4350)
    _sampled([f], [g], h, 1e-11, 4096)
    _poly_check([f], [g], h, 1e-11)


def test_config3_explicit_variant(ctx, H):
    d = synth.config_inputs(3)
    f, g = d["f"][0], d["g"][0]
    h = ctx.hd_conv_explicit([torch.from_numpy(f).cuda()], [torch.from_numpy(g).cuda()]).cpu().numpy()
    _sampled([f], [g], h, 1e-11, 1024)


def test_config4_full(ctx, H):
    d = synth.config_inputs(4)
    f, g = d["f"][0], d["g"][0]
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()).cpu().numpy()
    assert h.shape == (640, 640, 640) and h.dtype == np.complex64
    _sampled([f], [g], h, 1e-5, 192)
    _poly_check([f], [g], h.astype(np.complex128), 1e-5, npts=2)


def test_config5_full(ctx, H):
    d = synth.config_inputs(5)
    fs, gs = d["f"], d["g"]
    plan = ctx.tune(H.HD_C128, [2048, 2048], [1024, 1536], N=6, reps=2)
    h = ctx.multiconv([torch.from_numpy(a).cuda() for a in fs],
                      [torch.from_numpy(a).cuda() for a in gs], plan=plan).cpu().numpy()
    assert h.shape == (3071, 3583)
    _sampled(fs, gs, h, 1e-11, 256)
    _poly_check(fs, gs, h, 1e-11, npts=2)
