"""GPU parity of the multi-GPU entry points (include/hdconv.h "multi-GPU";
paper_2306_10016_b200/csrc/hd_dist.cu) against the oracle's direct convolution
(PAPER.md:537-541).  Only one GPU is available to these tests, so:
  * the NCCL path runs at world size 1 (hd_dist_init without a communicator) through
    the public entry points, including the chunked 2-D schedule (nchunks > 1);
  * several ranks are emulated with hd_slab_stage -- each rank's compute stages,
    the all-to-alls replaced by device block copies between the ranks' buffers
    (no kernel of one rank waits on another's);
  * residue sharding is checked as its definition: the partial convolutions over a
    partition of the residues (hd_pass r_begin / r_end) sum to the convolution."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import hdconv
    return hdconv


@pytest.fixture(scope="module")
def ctx(H):
    c = H.Context(0)
    assert c.dist_init() == (1, 0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def tol(dtype):
    return 1e-11 if dtype == np.complex128 else 1e-5


@pytest.mark.parametrize("Lf,Lg,m,nchunks", [((300, 260), (31, 17), (64, 64), 1),
                                             ((300, 260), (31, 17), (64, 64), 3),
                                             ((257, 4000), (20, 255), (128, 512), 4),   # x on the staged engine
                                             ((1100, 700), (255, 60), (512, 512), 2)])  # y conv q = 3 staged
def test_conv2d_dist_world1(ctx, H, Lf, Lg, m, nchunks):
    f, g = synth.random_pair(3000 + Lf[0], Lf, Lg)
    plan = H.Plan.make(2, [{"m": m[0]}, {"m": m[1]}])
    h = host(ctx.conv2d_dist(dev(f), dev(g), list(Lf), plan=plan, nchunks=nchunks))
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11


@pytest.mark.parametrize("dtype,m", [(np.complex128, 16), (np.complex64, 128)])
def test_conv3d_dist_world1(ctx, H, dtype, m):
    Lf, Lg = (150, 18, 24), (5, 7, 4)
    f, g = synth.random_pair(3100, Lf, Lg, dtype=dtype)
    plan = H.Plan.make(3, [{"m": m, "C": 4 if m == 128 else 1}] * 3)
    h = host(ctx.conv3d_dist(dev(f), dev(g), list(Lf), plan=plan))
    assert oracle.rel_l2(h, oracle.conv(f, g)) < tol(dtype)


@pytest.mark.parametrize("shard", [0, 1])
def test_conv1d_dist_world1(ctx, H, shard):
    B, Lf, Lg = 6, 3000, 700
    f, g = synth.random_pair(3200 + shard, (B, Lf), (B, Lg))
    h = host(ctx.conv1d_dist(dev(f), dev(g), B, shard=shard, plan=H.Plan.make(1, [{"m": 512}])))
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11


@pytest.mark.parametrize("shard", [0, 1])
def test_conv1d_dist_world1_default_plan_long_lines(ctx, H, shard):
    """config 2's line shape with the default plan (m = 4096, D = q = 3): batch sharding
    runs the one-CTA-per-line engine, residue sharding the generic pass with D lowered to
    what its shared memory holds."""
    B, Lf, Lg = 3, 8192, 3000
    f, g = synth.random_pair(3250 + shard, (B, Lf), (B, Lg))
    h = host(ctx.conv1d_dist(dev(f), dev(g), B, shard=shard))
    for b in range(B):
        assert oracle.rel_l2(h[b], oracle.conv(f[b], g[b])) < 1e-11


@pytest.mark.parametrize("q_parts", [[0, 1, 4, 7], [0, 3, 7], [0, 7]])
def test_residue_ranges_sum_to_the_convolution(ctx, H, q_parts):
    """hd_pass CONV over residues [r_begin, r_end): the partial backward sums over a
    partition of the q residues add up to the full convolution."""
    B, Lf, Lg, m = 3, 2500, 900, 512
    f, g = synth.random_pair(3300, (B, Lf), (B, Lg))
    fd, gd = dev(f), dev(g)
    Lout = Lf + Lg - 1
    q = -(-Lout // m)
    assert q == 7
    acc = np.zeros((B, Lout), dtype=np.complex128)
    for r0, r1 in zip(q_parts[:-1], q_parts[1:]):
        out = torch.empty((B, Lout), dtype=torch.complex128, device="cuda")
        d = H.PassDesc()
        d.mode, d.npairs, d.nlines, d.nbatch, d.M = H.HD_PASS_CONV, 1, B, 1, q * m
        d.axis.m, d.axis.C, d.axis.D = m, 1, 0
        d.in_f = H.Lines.make([fd.data_ptr()], Lf, s_l=Lf)
        d.in_g = H.Lines.make([gd.data_ptr()], Lg, s_l=Lg)
        d.out = H.Lines.make([out.data_ptr()], Lout, s_l=Lout)
        d.scale = 1.0 / (q * m)
        d.r_begin, d.r_end = r0, r1
        ctx.hd_pass(H.HD_C128, d)
        acc += host(out)
    for b in range(B):
        assert oracle.rel_l2(acc[b], oracle.conv(f[b], g[b])) < 1e-11
    bad = H.PassDesc()
    bad.mode, bad.npairs, bad.nlines, bad.nbatch, bad.M = H.HD_PASS_FWD, 1, B, 1, q * m
    bad.axis.m, bad.r_begin, bad.r_end = m, 1, 2
    bad.in_f = H.Lines.make([fd.data_ptr()], Lf, s_l=Lf)
    bad.out = H.Lines.make([fd.data_ptr()], q * m, s_l=q * m)
    with pytest.raises(H.HDError):
        ctx.hd_pass(H.HD_C128, bad)


def _emulate(ctx, H, dt, Lf, Lg, f, g, world, nchunks, plan):
    """Run every rank's stages with the all-to-alls as device block copies."""
    tdt = torch.complex128 if dt == H.HD_C128 else torch.complex64
    sps = [H.slab_plan(dt, Lf, Lg, world, k, nchunks, plan) for k in range(world)]
    el = [H.slab_buffer_elems(dt, sp, Lf, Lg) for sp in sps]
    new = lambda n: torch.zeros(max(int(n), 1), dtype=tdt, device="cuda")  # noqa: E731
    gd = dev(g)
    gts, s1 = [], []
    for k, sp in enumerate(sps):
        gt, sc = new(el[k]["g"]), new(el[k]["scratch"])
        ctx.slab_stage(dt, sp, Lf, Lg, 0, gd, gt, scratch=sc)
        out = new(el[k]["x1"])
        ctx.slab_stage(dt, sp, Lf, Lg, 1, dev(f[sp.in_lo:sp.in_hi]), out, scratch=sc)
        gts.append(gt)
        s1.append(out)

    def a2a(sends, block):
        recvs = [torch.zeros_like(s) for s in sends]
        for src in range(world):
            for dst in range(world):
                recvs[dst][src * block:(src + 1) * block] = sends[src][dst * block:(dst + 1) * block]
        return recvs

    def a2a_pieces(sends, block, P, C):
        """2-D exchanges (include/hdconv.h): send chunk-major, recv source-major."""
        recvs = [torch.zeros_like(s) for s in sends]
        for src in range(world):
            for dst in range(world):
                for c in range(C):
                    recvs[dst][src * block + c * P:src * block + (c + 1) * P] = \
                        sends[src][(c * world + dst) * P:(c * world + dst + 1) * P]
        return recvs
    sp0 = sps[0]
    two = len(Lf) == 2
    r1 = a2a_pieces(s1, sp0.block1, sp0.Ks * sp0.chunk_rows, sp0.nchunks) if two else a2a(s1, sp0.block1)
    s2 = []
    for k, sp in enumerate(sps):
        out = new(el[k]["x2"])
        ctx.slab_stage(dt, sp, Lf, Lg, 2, r1[k], out, gt=gts[k])
        s2.append(out)
    r2 = a2a_pieces(s2, sp0.block2, sp0.Ro * sp0.chunk_cols, sp0.nchunks) if two else a2a(s2, sp0.block2)
    parts = []
    for k, sp in enumerate(sps):
        O = [sp.out_hi - sp.out_lo] + [a + b - 1 for a, b in zip(Lf[1:], Lg[1:])]
        h = torch.empty(O, dtype=tdt, device="cuda")
        if sp.out_hi > sp.out_lo:
            ctx.slab_stage(dt, sp, Lf, Lg, 3, r2[k], h, scratch=new(el[k]["scratch"]))
        parts.append(host(h))
    return np.concatenate(parts, axis=0)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("Lf,Lg,m,nchunks", [((300, 260), (31, 17), (64, 64), 0),
                                             ((1100, 700), (255, 60), (512, 512), 3),
                                             ((257, 4000), (20, 255), (128, 512), 2),
                                             # pieces that tile the lines (1024 rows, 1024
                                             # spectral columns): the staged passes load
                                             # recv1 / recv2 by TMA_ELEM2 at worlds 2 and 4
                                             ((1024, 700), (255, 60), (512, 512), 2)])
def test_slab2d_emulated_ranks(ctx, H, world, Lf, Lg, m, nchunks):
    f, g = synth.random_pair(3400 + world, Lf, Lg)
    plan = H.Plan.make(2, [{"m": m[0]}, {"m": m[1]}])
    h = _emulate(ctx, H, H.HD_C128, list(Lf), list(Lg), f, g, world, nchunks, plan)
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype,m,C", [(np.complex128, 16, 1), (np.complex64, 16, 1), (np.complex64, 128, 4)])
def test_slab3d_emulated_ranks(ctx, H, world, dtype, m, C):
    Lf, Lg = (21, 18, 24) if m < 128 else (150, 18, 24), (5, 7, 4)
    f, g = synth.random_pair(3500 + world, Lf, Lg, dtype=dtype)
    dt = H.HD_C128 if dtype == np.complex128 else H.HD_C64
    plan = H.Plan.make(3, [{"m": m, "C": C}] * 3)
    n0 = ctx.engine_launches(H.HD_ENGINE_S128)
    h = _emulate(ctx, H, dt, list(Lf), list(Lg), f, g, world, 1, plan)
    assert oracle.rel_l2(h, oracle.conv(f, g)) < tol(dtype)
    if m == 128:  # kx tiles of 4: every pass of every rank on the staged engine
        assert ctx.engine_launches(H.HD_ENGINE_S128) - n0 == 7 * world
