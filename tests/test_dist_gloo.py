"""World-size-2 CPU test (gloo) of the slab-decomposition host logic
(paper_2306_10016_b200/dist.py): partitions, exchange layouts, padding of the
last slab.  The per-rank compute steps use a numpy stand-in backend with the SAME
buffer layouts as the GPU backend (natural frequency order, numpy FFT); the result
gathered from both ranks must equal the oracle's direct convolution."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2306_10016_b200.dist import SlabConv2D, SlabConv3D, SlabPlan2D, SlabPlan3D


class NumpyBackend:
    """Test stand-in for GpuBackend: same layouts, numpy transforms."""

    def __init__(self, Ky):
        self.Ky = Ky

    def empty(self, n):
        return np.zeros(max(1, n), dtype=np.complex128)

    def fwd_rows(self, f_rows, nrows, out, P):
        for y in range(nrows):
            X = np.fft.ifft(f_rows[y], n=P.Kx) * P.Kx            # + exponent, unnormalised
            for kx in range(P.Kx):
                out[(kx // P.Ks) * (P.Ks * P.R) + (kx % P.Ks) * P.R + y] = X[kx]

    def fwd_full(self, g, out, P):
        for y in range(P.Lg[0]):
            X = np.fft.ifft(g[y], n=P.Kx) * P.Kx
            out[np.arange(P.Kx) * P.Lg[0] + y] = X

    def conv_cols(self, xrecv, xg, ncols, col0, out, P):
        for c in range(ncols):
            ys = np.arange(P.Lf[0])
            fcol = xrecv[(ys // P.R) * (P.Ks * P.R) + c * P.R + ys % P.R]
            gcol = xg[(col0 + c) * P.Lg[0] + np.arange(P.Lg[0])]
            F = np.fft.ifft(fcol, n=self.Ky) * self.Ky
            G = np.fft.ifft(gcol, n=self.Ky) * self.Ky
            V = np.fft.fft(F * G) / (P.Kx * self.Ky)             # - exponent, scaled
            yo = np.arange(P.Oy)
            out[(yo // P.Ro) * (P.Ks * P.Ro) + (yo % P.Ro) * P.Ks + c] = V[: P.Oy]

    def inv_rows(self, yrecv, nrows, P):
        h = np.zeros((nrows, P.Ox), dtype=np.complex128)
        kx = np.arange(P.Kx)
        for y in range(nrows):
            row = yrecv[(kx // P.Ks) * (P.Ks * P.Ro) + y * P.Ks + kx % P.Ks]
            h[y] = np.fft.fft(row)[: P.Ox]
        return h


def gloo_exchange(send, recv, block):
    s = torch.view_as_real(torch.from_numpy(send))
    r = torch.view_as_real(torch.from_numpy(recv))
    n = dist.get_world_size()
    dist.all_to_all_single(r[: n * block], s[: n * block])


def _worker(rank, world, port, Lf, Lg, Kx, Ky, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f, g = synth.random_pair(321, Lf, Lg)
        P = SlabPlan2D(world, Lf, Lg, Kx)
        r0, r1 = P.rows(rank)
        conv = SlabConv2D(NumpyBackend(Ky), gloo_exchange, world, rank, Lf, Lg, Kx)
        h = conv(np.ascontiguousarray(f[r0:r1]), g)
        parts = [None] * world
        dist.all_gather_object(parts, h)
        if rank == 0:
            q.put(np.concatenate(parts, axis=0))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("Lf,Lg,Kx,Ky", [((13, 11), (4, 6), 20, 16), ((9, 7), (5, 5), 12, 13),
                                          ((8, 16), (1, 3), 18, 8)])
def test_slab_decomposition_two_ranks(Lf, Lg, Kx, Ky):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, Lf, Lg, Kx, Ky, q)) for r in range(world)]
    for p in procs:
        p.start()
    h = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f, g = synth.random_pair(321, Lf, Lg)
    ref = oracle.conv(f, g)
    assert h.shape == ref.shape
    assert oracle.rel_l2(h, ref) < 1e-12


def test_slab_plan_partitions():
    for world in (1, 2, 3, 4, 8):
        P = SlabPlan2D(world, (4096, 4096), (255, 255), 4608)
        rows = [P.rows(k) for k in range(world)]
        assert rows[0][0] == 0 and rows[-1][1] == 4096
        assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
        outs = [P.out_rows(k) for k in range(world)]
        assert outs[-1][1] == 4350 and sum(b - a for a, b in outs) == 4350
        cols = [P.cols(k) for k in range(world)]
        assert sum(b - a for a, b in cols) == 4608
        assert P.bytes_sent_per_rank(16) == (world - 1) * (P.x_block + P.y_block) * 16


# ---------------------------------------------------------------- 3-D z-slabs
class NumpyBackend3D:
    """Test stand-in for GpuBackend3D: same exchange layouts, numpy transforms."""

    def __init__(self, Kz):
        self.Kz = Kz

    def empty(self, n):
        return np.zeros(max(1, n), dtype=np.complex128)

    @staticmethod
    def _xy(planes, Ky, Kx):
        X = np.fft.ifft(planes, n=Kx, axis=2) * Kx                # + exponent, unnormalised
        return np.fft.ifft(X, n=Ky, axis=1) * Ky                  # [z][ky][kx]

    def fwd_planes(self, f_planes, nz, send, P):
        S = self._xy(f_planes, P.Ky, P.Kx)
        kx = np.arange(P.Kx)
        for zl in range(nz):
            for ky in range(P.Ky):
                send[P.ex1(ky // P.Kys, ky % P.Kys, kx, zl)] = S[zl, ky]

    def fwd_g(self, g, xyg, P):
        S = self._xy(g, P.Ky, P.Kx)                               # [z][ky][kx]
        xyg[: P.Ky * P.Kx * P.Lg[0]] = np.transpose(S, (1, 2, 0)).reshape(-1)

    def conv_lines(self, recv1, xyg, ky0, nky, send2, P):
        zs, zo = np.arange(P.Lf[0]), np.arange(P.O[0])
        for kyl in range(nky):
            for kx in range(P.Kx):
                fcol = recv1[P.ex1(zs // P.Rz, kyl, kx, zs % P.Rz)]
                gcol = xyg[((ky0 + kyl) * P.Kx + kx) * P.Lg[0] + np.arange(P.Lg[0])]
                F = np.fft.ifft(fcol, n=self.Kz) * self.Kz
                G = np.fft.ifft(gcol, n=self.Kz) * self.Kz
                V = np.fft.fft(F * G) / (self.Kz * P.Ky * P.Kx)
                send2[P.ex2(zo // P.Roz, zo % P.Roz, kx, kyl)] = V[: P.O[0]]

    def inv_planes(self, recv2, nzo, P):
        h = np.zeros((nzo, P.O[1], P.O[2]), dtype=np.complex128)
        ky = np.arange(P.Ky)
        for zol in range(nzo):
            W = np.zeros((P.O[1], P.Kx), dtype=np.complex128)
            for kx in range(P.Kx):
                row = recv2[P.ex2(ky // P.Kys, zol, kx, ky % P.Kys)]
                W[:, kx] = np.fft.fft(row)[: P.O[1]]
            h[zol] = np.fft.fft(W, axis=1)[:, : P.O[2]]
        return h


def _worker3d(rank, world, port, Lf, Lg, Kz, Ky, Kx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f, g = synth.random_pair(322, Lf, Lg)
        P = SlabPlan3D(world, Lf, Lg, Ky, Kx)
        z0, z1 = P.planes(rank)
        conv = SlabConv3D(NumpyBackend3D(Kz), gloo_exchange, world, rank, Lf, Lg, Ky, Kx)
        h = conv(np.ascontiguousarray(f[z0:z1]), g)
        parts = [None] * world
        dist.all_gather_object(parts, h)
        if rank == 0:
            q.put(np.concatenate(parts, axis=0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Lf,Lg,K", [((7, 6, 5), (3, 4, 2), (10, 12, 8)), ((4, 9, 6), (5, 2, 3), (9, 11, 9))])
def test_slab3d_two_ranks(Lf, Lg, K):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker3d, args=(r, world, port, Lf, Lg, K[0], K[1], K[2], q))
             for r in range(world)]
    for p in procs:
        p.start()
    h = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f, g = synth.random_pair(322, Lf, Lg)
    ref = oracle.conv(f, g)
    assert h.shape == ref.shape
    assert oracle.rel_l2(h, ref) < 1e-12


def test_slab3d_plan_partitions():
    for world in (1, 2, 3, 8):
        P = SlabPlan3D(world, (512, 512, 512), (129, 129, 129), 640, 640)
        pl = [P.planes(k) for k in range(world)]
        assert pl[0][0] == 0 and pl[-1][1] == 512 and all(pl[i][1] == pl[i + 1][0] for i in range(world - 1))
        assert sum(b - a for a, b in (P.out_planes(k) for k in range(world))) == 640
        assert sum(b - a for a, b in (P.kys(k) for k in range(world))) == 640
        assert P.bytes_sent_per_rank(8) == (world - 1) * (P.block1 + P.block2) * 8


def test_slab3d_exchange_layout_is_a_bijection():
    """ex1/ex2 place every (block, row, kx, plane) element once inside its block, with
    T = 4 consecutive kx adjacent (the tiled layouts GpuBackend3D describes to hd_pass)."""
    for world, K in ((1, (640, 640)), (3, (640, 640)), (2, (12, 9))):
        P = SlabPlan3D(world, (20, 7, 5), (5, 3, 2), *K)
        assert P.T == (4 if K[1] % 4 == 0 else 1)
        kyl, kx, zl = np.meshgrid(np.arange(P.Kys), np.arange(P.Kx), np.arange(P.Rz), indexing="ij")
        for blk in range(world):
            o = P.ex1(blk, kyl, kx, zl).ravel()
            assert np.array_equal(np.sort(o), blk * P.block1 + np.arange(P.block1))
        zol, kx2, kyl2 = np.meshgrid(np.arange(P.Roz), np.arange(P.Kx), np.arange(P.Kys), indexing="ij")
        for blk in range(world):
            o = P.ex2(blk, zol, kx2, kyl2).ravel()
            assert np.array_equal(np.sort(o), blk * P.block2 + np.arange(P.block2))
        if P.T == 4:
            assert P.ex1(0, 0, 1, 0) - P.ex1(0, 0, 0, 0) == 1 and P.ex2(0, 0, 3, 0) - P.ex2(0, 0, 0, 0) == 3
