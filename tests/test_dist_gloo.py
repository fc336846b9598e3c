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
from paper_2306_10016_b200.dist import SlabConv2D, SlabPlan2D


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
            out[(yo // P.Ro) * (P.Ks * P.Ro) + c * P.Ro + yo % P.Ro] = V[: P.Oy]

    def inv_rows(self, yrecv, nrows, P):
        h = np.zeros((nrows, P.Ox), dtype=np.complex128)
        kx = np.arange(P.Kx)
        for y in range(nrows):
            row = yrecv[(kx // P.Ks) * (P.Ks * P.Ro) + (kx % P.Ks) * P.Ro + y]
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
