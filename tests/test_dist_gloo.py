"""World-size-2 CPU tests (gloo) of the slab decomposition's host logic in
libhdconv.so (hd_dist_slab_plan, hd_dist_partition: include/hdconv.h "multi-GPU").

The layouts the library's passes read and write (paper_2306_10016_b200/csrc/
hd_dist.cu, comments above slab2d_stage / slab3d_stage) are restated here as a
numpy model driven by the C plan's numbers (rows, output rows, spectral lines,
chunk sizes, block sizes, normalisation); two gloo ranks run the model with real
all-to-alls and the gathered result must equal the oracle's direct convolution
(PAPER.md:537-541).  The GPU side of the same layouts is covered by the
emulated-rank tests in tests/test_gpu_dist.py (hd_slab_stage)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import hdconv
    return hdconv


def _plan(H, ndim, m):
    return H.Plan.make(ndim, [{"m": mm} for mm in m])


class Model2D:
    """numpy stand-in of the four 2-D stages (natural frequency order, numpy FFT)."""

    def __init__(self, sp, Lf, Lg):
        self.sp, self.Lf, self.Lg = sp, Lf, Lg
        self.Ky, self.Kx = sp.plan.axis[0].M1, sp.plan.axis[1].M1
        self.Oy, self.Ox = Lf[0] + Lg[0] - 1, Lf[1] + Lg[1] - 1

    def stage0(self, g):
        xg = np.zeros(self.Kx * self.Lg[0], dtype=np.complex128)
        for y in range(self.Lg[0]):
            xg[np.arange(self.Kx) * self.Lg[0] + y] = np.fft.ifft(g[y], n=self.Kx) * self.Kx
        return xg

    def stage1(self, f_rows):
        """send1 [row chunk][kx / 16][y % Rc][kx % 16] (chunk-major, 16-wide kx tiles)."""
        sp = self.sp
        Rc = sp.chunk_rows
        out = np.zeros(sp.nranks * sp.block1, dtype=np.complex128)
        kx = np.arange(self.Kx)
        for yl in range(sp.in_hi - sp.in_lo):
            c, yi = divmod(yl, Rc)
            X = np.fft.ifft(f_rows[yl], n=self.Kx) * self.Kx       # + exponent, unnormalised
            out[c * sp.nranks * sp.Ks * Rc + (kx // 16) * (16 * Rc) + yi * 16 + kx % 16] = X
        return out

    def stage2(self, recv1, xg):
        sp = self.sp
        out = np.zeros(sp.nranks * sp.block2, dtype=np.complex128)
        ys, yo = np.arange(self.Lf[0]), np.arange(self.Oy)
        for c in range(sp.spec_hi - sp.spec_lo):
            cc, ci = divmod(c, sp.chunk_cols)
            kx = sp.spec_lo + c
            Rc = sp.chunk_rows
            fcol = recv1[(ys // Rc) * (sp.Ks * Rc) + (c // 16) * (16 * Rc) + (ys % Rc) * 16 + c % 16]
            gcol = xg[kx * self.Lg[0] + np.arange(self.Lg[0])]
            F = np.fft.ifft(fcol, n=self.Ky) * self.Ky
            G = np.fft.ifft(gcol, n=self.Ky) * self.Ky
            V = np.fft.fft(F * G) * sp.scale                        # - exponent, 1 / (M1_y M1_x)
            Kc = sp.chunk_cols       # send2 [chunk][yo][kx % Kc] (chunk-major)
            out[cc * sp.nranks * sp.Ro * Kc + yo * Kc + ci] = V[: self.Oy]
        return out

    def stage3(self, recv2):
        sp = self.sp
        h = np.zeros((sp.out_hi - sp.out_lo, self.Ox), dtype=np.complex128)
        kx = np.arange(self.Kx)
        Kc = sp.chunk_cols
        for yl in range(sp.out_hi - sp.out_lo):
            row = recv2[(kx // Kc) * (sp.Ro * Kc) + yl * Kc + kx % Kc]
            h[yl] = np.fft.fft(row)[: self.Ox]
        return h


class Model3D:
    """numpy stand-in of the four 3-D stages (layouts of hd_dist.cu slab3d_stage)."""

    def __init__(self, sp, Lf, Lg):
        self.sp, self.Lf, self.Lg = sp, Lf, Lg
        self.Kz, self.Ky, self.Kx = (sp.plan.axis[i].M1 for i in range(3))
        self.O = tuple(a + b - 1 for a, b in zip(Lf, Lg))
        self.T = sp.chunk_cols

    def ex1(self, blk, kyl, kx, zl):
        sp, T = self.sp, self.T
        return blk * sp.block1 + kyl * (self.Kx * sp.R) + (kx // T) * (sp.R * T) + zl * T + kx % T

    def ex2(self, blk, zol, kx, kyl):
        sp, T = self.sp, self.T
        return blk * sp.block2 + zol * (self.Kx * sp.Ks) + (kx // T) * (sp.Ks * T) + kyl * T + kx % T

    def _xy(self, planes):
        X = np.fft.ifft(planes, n=self.Kx, axis=2) * self.Kx
        return np.fft.ifft(X, n=self.Ky, axis=1) * self.Ky       # [z][ky][kx]

    def stage0(self, g):
        return np.transpose(self._xy(g), (1, 2, 0)).reshape(-1)  # [ky][kx][z]

    def stage1(self, f_planes):
        sp = self.sp
        out = np.zeros(sp.nranks * sp.block1, dtype=np.complex128)
        if sp.in_hi > sp.in_lo:
            S = self._xy(f_planes)
            kx = np.arange(self.Kx)
            for zl in range(sp.in_hi - sp.in_lo):
                for ky in range(self.Ky):
                    out[self.ex1(ky // sp.Ks, ky % sp.Ks, kx, zl)] = S[zl, ky]
        return out

    def stage2(self, recv1, xyg):
        sp = self.sp
        out = np.zeros(sp.nranks * sp.block2, dtype=np.complex128)
        zs, zo = np.arange(self.Lf[0]), np.arange(self.O[0])
        for kyl in range(sp.spec_hi - sp.spec_lo):
            for kx in range(self.Kx):
                fcol = recv1[self.ex1(zs // sp.R, kyl, kx, zs % sp.R)]
                gcol = xyg[((sp.spec_lo + kyl) * self.Kx + kx) * self.Lg[0] + np.arange(self.Lg[0])]
                F = np.fft.ifft(fcol, n=self.Kz) * self.Kz
                G = np.fft.ifft(gcol, n=self.Kz) * self.Kz
                V = np.fft.fft(F * G) * sp.scale
                out[self.ex2(zo // sp.Ro, zo % sp.Ro, kx, kyl)] = V[: self.O[0]]
        return out

    def stage3(self, recv2):
        sp = self.sp
        h = np.zeros((sp.out_hi - sp.out_lo, self.O[1], self.O[2]), dtype=np.complex128)
        ky = np.arange(self.Ky)
        for zol in range(sp.out_hi - sp.out_lo):
            W = np.zeros((self.O[1], self.Kx), dtype=np.complex128)
            for kx in range(self.Kx):
                W[:, kx] = np.fft.fft(recv2[self.ex2(ky // sp.Ks, zol, kx, ky % sp.Ks)])[: self.O[1]]
            h[zol] = np.fft.fft(W, axis=1)[:, : self.O[2]]
        return h


def _exchange(send, block):
    recv = np.zeros_like(send)
    s = torch.view_as_real(torch.from_numpy(send))
    r = torch.view_as_real(torch.from_numpy(recv))
    dist.all_to_all_single(r, s)
    return recv


def _exchange_2d(send, block, P, sp):
    """A 2-D exchange (include/hdconv.h): per chunk c, the pieces of P elements for
    every rank (chunk-major in send) go to source-major slots (block, c) of recv."""
    C, n = sp.nchunks, sp.nranks
    recv = np.zeros_like(send)
    for c in range(C):
        tmp = np.zeros(n * P, dtype=send.dtype)
        s = torch.view_as_real(torch.from_numpy(np.ascontiguousarray(send[c * n * P:(c + 1) * n * P])))
        dist.all_to_all_single(torch.view_as_real(torch.from_numpy(tmp)), s)
        for src in range(n):
            recv[src * block + c * P:src * block + (c + 1) * P] = tmp[src * P:(src + 1) * P]
    return recv


def _worker(rank, world, port, ndim, Lf, Lg, m, nchunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_10016_b200 import hdconv as H
        f, g = synth.random_pair(321 + ndim, Lf, Lg)
        sp = H.slab_plan(H.HD_C128, Lf, Lg, world, rank, nchunks, _plan(H, ndim, m))
        M = (Model2D if ndim == 2 else Model3D)(sp, Lf, Lg)
        gt = M.stage0(g)
        s1 = M.stage1(np.ascontiguousarray(f[sp.in_lo:sp.in_hi]))
        if ndim == 2:
            r1 = _exchange_2d(s1, sp.block1, sp.Ks * sp.chunk_rows, sp)
            r2 = _exchange_2d(M.stage2(r1, gt), sp.block2, sp.Ro * sp.chunk_cols, sp)
        else:
            r1 = _exchange(s1, sp.block1)
            r2 = _exchange(M.stage2(r1, gt), sp.block2)
        h = M.stage3(r2)
        parts = [None] * world
        dist.all_gather_object(parts, (sp.out_lo, h))
        if rank == 0:
            q.put(np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])], axis=0))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(ndim, Lf, Lg, m, nchunks, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ndim, Lf, Lg, m, nchunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    h = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f, g = synth.random_pair(321 + ndim, Lf, Lg)
    ref = oracle.conv(f, g)
    assert h.shape == ref.shape
    assert oracle.rel_l2(h, ref) < 1e-12


@pytest.mark.parametrize("Lf,Lg,m,nchunks", [((13, 11), (4, 6), (4, 8), 0), ((9, 7), (5, 5), (8, 4), 3),
                                             ((8, 16), (1, 3), (4, 4), 1), ((21, 10), (6, 3), (16, 8), 4)])
def test_slab2d_two_ranks(Lf, Lg, m, nchunks):
    _run(2, Lf, Lg, m, nchunks)


@pytest.mark.parametrize("Lf,Lg,m", [((7, 6, 5), (3, 4, 2), (4, 4, 4)), ((4, 9, 6), (5, 2, 3), (8, 4, 2))])
def test_slab3d_two_ranks(Lf, Lg, m):
    _run(3, Lf, Lg, m, 1)


def test_partition_covers(H):
    for extent in (0, 1, 7, 4096, 4350):
        for world in (1, 2, 3, 8):
            parts = [H.dist_partition(extent, world, k) for k in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == extent
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def test_slab2d_plan_config3(H):
    """Config 3 (4096^2 * 255^2, m = 512): every rank's rows, output rows and spectral
    columns tile the problem; chunks divide the padded slabs; the bytes each rank
    sends are the two blocks to every other rank; scale = 1 / (M1_y M1_x)."""
    for world in (1, 2, 3, 4, 8):
        sps = [H.slab_plan(H.HD_C128, [4096, 4096], [255, 255], world, k) for k in range(world)]
        s0 = sps[0]
        assert s0.nchunks == (2 if world > 1 else 1)
        assert s0.R == s0.nchunks * s0.chunk_rows and s0.Ks == s0.nchunks * s0.chunk_cols
        assert s0.R * world >= 4096 and s0.Ro * world >= 4350 and s0.Ks * world >= 4608
        for key, n in (("in", 4096), ("out", 4350), ("spec", 4608)):
            lo = [getattr(s, key + "_lo") for s in sps]
            hi = [getattr(s, key + "_hi") for s in sps]
            assert lo[0] == 0 and hi[-1] == n and all(hi[i] == lo[i + 1] for i in range(world - 1))
        assert s0.block1 == s0.Ks * s0.R and s0.block2 == s0.Ks * s0.Ro
        assert s0.bytes_sent == (world - 1) * (s0.block1 + s0.block2) * 16
        assert s0.scale == pytest.approx(1.0 / (s0.plan.axis[0].M1 * s0.plan.axis[1].M1))


def test_slab3d_plan_config4(H):
    for world in (1, 2, 3, 8):
        sps = [H.slab_plan(H.HD_C64, [512] * 3, [129] * 3, world, k) for k in range(world)]
        s0 = sps[0]
        Ky, Kx = s0.plan.axis[1].M1, s0.plan.axis[2].M1
        assert s0.chunk_cols == (4 if Kx % 4 == 0 else 1)
        assert sum(s.in_hi - s.in_lo for s in sps) == 512
        assert sum(s.out_hi - s.out_lo for s in sps) == 640
        assert sum(s.spec_hi - s.spec_lo for s in sps) == Ky
        assert s0.block1 == s0.Ks * Kx * s0.R and s0.block2 == s0.Ks * Kx * s0.Ro
        assert s0.bytes_sent == (world - 1) * (s0.block1 + s0.block2) * 8


def test_slab2d_layout_is_a_bijection(H):
    """The chunked 2-D layouts place every (row, kx) and (output row, kx) element once."""
    for world, nch in ((1, 1), (2, 3), (3, 4)):
        sp = H.slab_plan(H.HD_C128, [21, 10], [6, 3], world, 0, nch, _plan(H, 2, (16, 8)))
        Kc, Rc = sp.chunk_cols, sp.chunk_rows
        yl, kx = np.meshgrid(np.arange(sp.R), np.arange(world * sp.Ks), indexing="ij")
        o1 = (kx // sp.Ks) * sp.block1 + (yl // Rc) * sp.Ks * Rc + (kx % sp.Ks) * Rc + yl % Rc
        assert np.array_equal(np.sort(o1.ravel()), np.arange(world * sp.block1))
        yo, c = np.meshgrid(np.arange(world * sp.Ro), np.arange(sp.Ks), indexing="ij")
        o2 = (yo // sp.Ro) * sp.block2 + (c // Kc) * sp.Ro * Kc + (yo % sp.Ro) * Kc + c % Kc
        assert np.array_equal(np.sort(o2.ravel()), np.arange(world * sp.block2))
