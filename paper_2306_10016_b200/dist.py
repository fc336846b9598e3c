"""Multi-GPU hybrid-dealiased 2D convolution by slab decomposition.

SURVEY §8(e): rank k holds a contiguous slab of f's rows (g is replicated);
  1. forward along x of the local rows (pass A)       -> X[dest][kx_local][y_local]
  2. all-to-all (exchange 1): rank k' receives the spectral columns of its slab
  3. convolution along y of the local columns (pass B) -> Y[dest][yo_local][kx_local]
     (row-major blocks: pass C then reads contiguous runs of every output row; the
     compute-bound pass B absorbs the strided stores)
  4. all-to-all (exchange 2): rank k receives its output rows for every column
  5. inverse along x of the local output rows (pass C) -> h rows
Every arithmetic step runs in libhdconv.so (`hd_pass`); this module only computes
partitions and layouts (plain integers) and calls the caller's all-to-all, which is
`torch.distributed.all_to_all_single` (NCCL over NVLink) in production.  The
layouts make every per-destination block contiguous, so the exchange needs no
packing.  The partition/exchange logic is shared with a CPU test backend
(tests/test_dist_gloo.py) that runs it on 2 gloo ranks.
"""
from __future__ import annotations

from dataclasses import dataclass


def cdiv(a, b):
    return -(-a // b)


@dataclass
class SlabPlan2D:
    """Partition of a 2D problem f [Lf0][Lf1] * g [Lg0][Lg1] over `world` ranks.
    Kx = M1 along x (spectral columns), Oy/Ox the output extents."""
    world: int
    Lf: tuple
    Lg: tuple
    Kx: int

    def __post_init__(self):
        self.Oy = self.Lf[0] + self.Lg[0] - 1
        self.Ox = self.Lf[1] + self.Lg[1] - 1
        self.R = cdiv(self.Lf[0], self.world)     # f rows per rank
        self.Ro = cdiv(self.Oy, self.world)       # output rows per rank
        self.Ks = cdiv(self.Kx, self.world)       # spectral columns per rank

    def rows(self, k):
        return k * self.R, min((k + 1) * self.R, self.Lf[0])

    def out_rows(self, k):
        return min(k * self.Ro, self.Oy), min((k + 1) * self.Ro, self.Oy)

    def cols(self, k):
        return min(k * self.Ks, self.Kx), min((k + 1) * self.Ks, self.Kx)

    # element counts of the exchange buffers (all per-destination blocks equal)
    @property
    def x_block(self):
        return self.Ks * self.R

    @property
    def y_block(self):
        return self.Ks * self.Ro

    def bytes_sent_per_rank(self, elem_bytes):
        """Bytes leaving one rank in the two exchanges (block to itself excluded)."""
        return (self.world - 1) * (self.x_block + self.y_block) * elem_bytes


class SlabConv2D:
    """Slab-decomposed 2D convolution on one rank of `world`.

    backend: object with
      fwd_rows(x_rows, nrows, Lx, out, plan)            pass A on local rows
      fwd_full(g, out)                                   pass A on the replicated g
      conv_cols(xrecv, xg, ncols, col0, out, plan)       pass B on local columns
      inv_rows(yrecv, nrows, out_rows, plan)             pass C on local output rows
      empty(n) -> buffer of n complex elements
    exchange(send, recv, block): all-to-all of `world` equal blocks of `block` elements.
    """

    def __init__(self, backend, exchange, world, rank, Lf, Lg, Kx):
        self.b = backend
        self.exchange = exchange
        self.rank = rank
        self.plan = SlabPlan2D(world, tuple(Lf), tuple(Lg), Kx)

    # the three compute stages between the two exchanges
    def stage1(self, f_rows, g):
        P, k, b = self.plan, self.rank, self.b
        r0, r1 = P.rows(k)
        xsend = b.empty(P.world * P.x_block)
        b.fwd_rows(f_rows, r1 - r0, xsend, P)
        xg = b.empty(P.Kx * P.Lg[0])
        b.fwd_full(g, xg, P)
        return xsend, xg

    def stage2(self, xrecv, xg):
        P, k, b = self.plan, self.rank, self.b
        c0, c1 = P.cols(k)
        ysend = b.empty(P.world * P.y_block)
        b.conv_cols(xrecv, xg, c1 - c0, c0, ysend, P)
        return ysend

    def stage3(self, yrecv):
        P, k = self.plan, self.rank
        o0, o1 = P.out_rows(k)
        return self.b.inv_rows(yrecv, o1 - o0, P)

    def __call__(self, f_rows, g):
        P, b = self.plan, self.b
        xsend, xg = self.stage1(f_rows, g)
        xrecv = b.empty(P.world * P.x_block)
        self.exchange(xsend, xrecv, P.x_block)
        ysend = self.stage2(xrecv, xg)
        yrecv = b.empty(P.world * P.y_block)
        self.exchange(ysend, yrecv, P.y_block)
        return self.stage3(yrecv)


def emulate_ranks(convs, f, g, empty):
    """Run `world` SlabConv2D instances in one process (test/validation tool): the
    all-to-all is replaced by block copies between the ranks' buffers."""
    world = len(convs)
    P = convs[0].plan
    xs = []
    for k, c in enumerate(convs):
        r0, r1 = P.rows(k)
        xs.append(c.stage1(f[r0:r1], g))
    def a2a(sends, block):
        recvs = [empty(world * block) for _ in range(world)]
        for src in range(world):
            for dst in range(world):
                recvs[dst][src * block:(src + 1) * block] = sends[src][dst * block:(dst + 1) * block]
        return recvs
    xr = a2a([x for x, _ in xs], P.x_block)
    ys = [c.stage2(xr[k], xs[k][1]) for k, c in enumerate(convs)]
    yr = a2a(ys, P.y_block)
    return [c.stage3(yr[k]) for k, c in enumerate(convs)]


class GpuBackend:
    """Passes on libhdconv.so through hd_pass descriptors (device tensors)."""

    def __init__(self, ctx, plan, dtype):
        import torch
        from . import hdconv as H
        self.H, self.torch, self.ctx = H, torch, ctx
        self.dt = dtype
        self.tdt = torch.complex128 if dtype == H.HD_C128 else torch.complex64
        p = plan.as_dict()["axis"]
        self.ax = p           # [y, x] completed axis plans (m, q, M1, C, D, threads)
        self.scale = 1.0 / (p[0]["M1"] * p[1]["M1"])
        self.dev = torch.device("cuda", torch.cuda.current_device())
        # the x passes (forward of f and g rows, inverse of the output rows) on the staged
        # m = 512 engine in its own spectral order when every one of them qualifies
        x = p[1]
        self.x_flags = (H.HD_FLAG_STAGED_ORDER
                        if dtype == H.HD_C128 and x["m"] == 512 and x["q"] <= 11 and x["p_f"] <= 8
                        and x["p_g"] <= 8 else 0)

    def empty(self, n):
        return self.torch.empty(max(1, n), dtype=self.tdt, device=self.dev)

    def _desc(self, mode, axis, nlines, M):
        H = self.H
        d = H.PassDesc()
        d.mode, d.npairs, d.nlines, d.nbatch, d.M = mode, 1, nlines, 1, M
        a = self.ax[axis]
        d.axis.m, d.axis.C, d.axis.D, d.axis.threads = a["m"], 1, 0, 0
        if axis == 1:
            d.flags = self.x_flags
        return d

    def fwd_rows(self, f_rows, nrows, out, P):
        if nrows <= 0:
            return
        H = self.H
        d = self._desc(H.HD_PASS_FWD, 1, nrows, self.ax[1]["M1"])
        d.in_f = H.Lines.make([f_rows.data_ptr()], P.Lf[1], s_l=P.Lf[1])
        # element kx of local row y -> (kx / Ks)*(Ks*R) + (kx % Ks)*R + y
        d.out = H.Lines.make([out.data_ptr()], P.Kx, s_l=1, s_j=P.R, jd=P.Ks, s_jt=P.Ks * P.R)
        self.ctx.hd_pass(self.dt, d)

    def fwd_full(self, g, out, P):
        H = self.H
        d = self._desc(H.HD_PASS_FWD, 1, P.Lg[0], self.ax[1]["M1"])
        d.in_f = H.Lines.make([g.data_ptr()], P.Lg[1], s_l=P.Lg[1])
        d.out = H.Lines.make([out.data_ptr()], P.Kx, s_l=1, s_j=P.Lg[0])   # X_g[kx][y]
        self.ctx.hd_pass(self.dt, d)

    def conv_cols(self, xrecv, xg, ncols, col0, out, P):
        if ncols <= 0:
            return
        H = self.H
        d = self._desc(H.HD_PASS_CONV, 0, ncols, self.ax[0]["M1"])
        d.in_f = H.Lines.make([xrecv.data_ptr()], P.Lf[0], s_l=P.R, s_j=1, jd=P.R, s_jt=P.Ks * P.R)
        eb = xg.element_size()
        d.in_g = H.Lines.make([xg.data_ptr() + col0 * P.Lg[0] * eb], P.Lg[0], s_l=P.Lg[0])
        # output row yo of local column c -> (yo / Ro)*(Ks*Ro) + (yo % Ro)*Ks + c
        # (lines as tiles of width 1: TMA can store the 16-byte pieces when one block
        #  holds every output row, i.e. Ro >= Oy)
        d.out = H.Lines.make([out.data_ptr()], P.Oy, s_l=1, s_j=P.Ks, jd=P.Ro, s_jt=P.Ks * P.Ro, tl=0, s_t=1)
        d.scale = self.scale
        self.ctx.hd_pass(self.dt, d)

    def inv_rows(self, yrecv, nrows, P):
        h = self.torch.empty((max(nrows, 0), P.Ox), dtype=self.tdt, device=self.dev)
        if nrows <= 0:
            return h
        H = self.H
        d = self._desc(H.HD_PASS_INV, 1, nrows, self.ax[1]["M1"])
        # element kx of local output row y -> (kx / Ks)*(Ks*Ro) + y*Ks + kx % Ks
        d.in_f = H.Lines.make([yrecv.data_ptr()], P.Kx, s_l=P.Ks, s_j=1, jd=P.Ks, s_jt=P.Ks * P.Ro)
        d.out = H.Lines.make([h.data_ptr()], P.Ox, s_l=P.Ox)
        self.ctx.hd_pass(self.dt, d)
        return h


# ---------------------------------------------------------------------------
# 3-D: z-slabs: rank k holds f planes [k Rz, (k+1) Rz) (g replicated)
#   1. forward along x, then y, of the local planes       -> send1[dest][kyl][kx][zl]
#   2. all-to-all: rank k' receives the spectral rows ky of its slab for every z
#   3. convolution along z of its (ky, kx) lines            -> send2[dest][kyl][kx][zol]
#   4. all-to-all: rank k receives its output planes for every (ky, kx)
#   5. inverse along y, then x, of the local output planes  -> h planes
@dataclass
class SlabPlan3D:
    """Partition of a 3-D problem f [Lf0][Lf1][Lf2] * g over `world` ranks; Ky, Kx the
    spectral extents (M1) along y and x."""
    world: int
    Lf: tuple
    Lg: tuple
    Ky: int
    Kx: int

    def __post_init__(self):
        self.O = tuple(a + b - 1 for a, b in zip(self.Lf, self.Lg))
        self.Rz = cdiv(self.Lf[0], self.world)      # f planes per rank
        self.Roz = cdiv(self.O[0], self.world)      # output planes per rank
        self.Kys = cdiv(self.Ky, self.world)        # spectral y rows per rank

    def planes(self, k):
        return min(k * self.Rz, self.Lf[0]), min((k + 1) * self.Rz, self.Lf[0])

    def out_planes(self, k):
        return min(k * self.Roz, self.O[0]), min((k + 1) * self.Roz, self.O[0])

    def kys(self, k):
        return min(k * self.Kys, self.Ky), min((k + 1) * self.Kys, self.Ky)

    @property
    def T(self):
        """kx tile of the exchange blocks: T consecutive kx of one (ky, z) are adjacent,
        so a pass over kx lines in groups of T moves T-element pieces (the 3-D
        pipeline's tiled layouts)."""
        return 4 if self.Kx % 4 == 0 else 1

    def ex1(self, blk, kyl, kx, zl):
        """Element offset in the first exchange buffer: block `blk` (destination ky
        range on the sender, source z slab on the receiver) [kyl][kx/T][zl][kx%T]."""
        T = self.T
        return blk * self.block1 + kyl * (self.Kx * self.Rz) + (kx // T) * (self.Rz * T) + zl * T + kx % T

    def ex2(self, blk, zol, kx, kyl):
        """Element offset in the second exchange buffer: block `blk` (destination z
        range on the sender, source ky range on the receiver) [zol][kx/T][kyl][kx%T]."""
        T = self.T
        return blk * self.block2 + zol * (self.Kx * self.Kys) + (kx // T) * (self.Kys * T) + kyl * T + kx % T

    @property
    def block1(self):
        return self.Kys * self.Kx * self.Rz

    @property
    def block2(self):
        return self.Kys * self.Kx * self.Roz

    def bytes_sent_per_rank(self, elem_bytes):
        return (self.world - 1) * (self.block1 + self.block2) * elem_bytes


class SlabConv3D:
    """Slab-decomposed 3-D convolution on one rank of `world`.

    backend: fwd_planes(f_planes, nz, send1, P)     passes 1 (x, then y) of the local planes
             fwd_g(g, xyg, P)                        the replicated g's x and y transforms
             conv_lines(recv1, xyg, ky0, nky, send2, P)  convolution along z
             inv_planes(recv2, nzo, P) -> h planes   passes 5 (y, then x)
             empty(n)
    exchange(send, recv, block) as for SlabConv2D."""

    def __init__(self, backend, exchange, world, rank, Lf, Lg, Ky, Kx):
        self.b = backend
        self.exchange = exchange
        self.rank = rank
        self.plan = SlabPlan3D(world, tuple(Lf), tuple(Lg), Ky, Kx)

    def stage1(self, f_planes, g):
        P, k, b = self.plan, self.rank, self.b
        z0, z1 = P.planes(k)
        send = b.empty(P.world * P.block1)
        b.fwd_planes(f_planes, z1 - z0, send, P)
        xyg = b.empty(P.Ky * P.Kx * P.Lg[0])
        b.fwd_g(g, xyg, P)
        return send, xyg

    def stage2(self, recv1, xyg):
        P, k, b = self.plan, self.rank, self.b
        y0, y1 = P.kys(k)
        send = b.empty(P.world * P.block2)
        b.conv_lines(recv1, xyg, y0, y1 - y0, send, P)
        return send

    def stage3(self, recv2):
        P, k = self.plan, self.rank
        o0, o1 = P.out_planes(k)
        return self.b.inv_planes(recv2, o1 - o0, P)

    def __call__(self, f_planes, g):
        P, b = self.plan, self.b
        s1, xyg = self.stage1(f_planes, g)
        r1 = b.empty(P.world * P.block1)
        self.exchange(s1, r1, P.block1)
        s2 = self.stage2(r1, xyg)
        r2 = b.empty(P.world * P.block2)
        self.exchange(s2, r2, P.block2)
        return self.stage3(r2)


def emulate_ranks_3d(convs, f, g, empty):
    """SlabConv3D on `world` emulated ranks in one process (block copies for the
    all-to-alls)."""
    world = len(convs)
    P = convs[0].plan
    st1 = []
    for k, c in enumerate(convs):
        z0, z1 = P.planes(k)
        st1.append(c.stage1(f[z0:z1], g))

    def a2a(sends, block):
        recvs = [empty(world * block) for _ in range(world)]
        for src in range(world):
            for dst in range(world):
                recvs[dst][src * block:(src + 1) * block] = sends[src][dst * block:(dst + 1) * block]
        return recvs
    r1 = a2a([s for s, _ in st1], P.block1)
    s2 = [c.stage2(r1[k], st1[k][1]) for k, c in enumerate(convs)]
    r2 = a2a(s2, P.block2)
    return [c.stage3(r2[k]) for k, c in enumerate(convs)]


class GpuBackend3D:
    """3-D slab passes on libhdconv.so (hd_pass descriptors, device tensors), in the
    3-D pipeline's tiled layouts (hd_api.cu run_pipeline, ndim 3): kx tiles of T = 4
    lines, so complex64 axes with m = 128 run on the staged engine (hd_s128.cuh; the
    forward/inverse passes with HD_FLAG_STAGED_ORDER, the same on both sides)."""

    def __init__(self, ctx, plan, dtype):
        import torch
        from . import hdconv as H
        self.H, self.torch, self.ctx = H, torch, ctx
        self.dt = dtype
        self.tdt = torch.complex128 if dtype == H.HD_C128 else torch.complex64
        self.ax = plan.as_dict()["axis"]     # [z, y, x]
        self.scale = 1.0 / (self.ax[0]["M1"] * self.ax[1]["M1"] * self.ax[2]["M1"])
        self.dev = torch.device("cuda", torch.cuda.current_device())

    def empty(self, n):
        return self.torch.empty(max(1, n), dtype=self.tdt, device=self.dev)

    def _staged(self, axis):
        """hd_s128.cuh's conditions for every pass along `axis` (api use_s128)."""
        a = self.ax[axis]
        return self.dt == self.H.HD_C64 and a["m"] == 128 and a["q"] <= 8 and max(a["p_f"], a["p_g"]) <= 8

    def _desc(self, mode, axis, nlines, nbatch, T):
        d = self.H.PassDesc()
        a = self.ax[axis]
        d.mode, d.npairs, d.nlines, d.nbatch, d.M = mode, 1, nlines, nbatch, a["M1"]
        staged = T == 4 and self._staged(axis)
        d.axis.m, d.axis.C, d.axis.D, d.axis.threads = a["m"], 4 if staged else 1, 0, 0
        if staged and mode != self.H.HD_PASS_CONV:
            d.flags = self.H.HD_FLAG_STAGED_ORDER
        return d

    @staticmethod
    def _lt(T, s_t):
        """line l at (l / T) * s_t + l % T (plain stride s_t when T = 1)."""
        return dict(tl=T.bit_length() - 1, s_t=s_t, s_l=1) if T > 1 else dict(s_l=s_t)

    @staticmethod
    def _et(T, s_jt, s_l):
        """line stride s_l, element j at (j / T) * s_jt + j % T (plain when T = 1)."""
        return dict(s_l=s_l, s_j=1, jd=T, s_jt=s_jt) if T > 1 else dict(s_l=s_l, s_j=s_jt)

    def _xy(self, src, nz, Ly, Lx, out_ptr, s_ky, s_t, s_z, T, jd=0, s_jt=0):
        """x then y forward transforms of nz planes [z][y][x]; spectral element (z, ky, kx)
        -> out + (ky tiling) + (kx / T) * s_t + kx % T + z * s_z."""
        H = self.H
        Kx = self.ax[2]["M1"]
        x1 = self.empty(nz * Kx * Ly)                                 # X1[z][kx/T][y][kx%T]
        d = self._desc(H.HD_PASS_FWD, 2, Ly, nz, T)
        d.in_f = H.Lines.make([src.data_ptr()], Lx, s_l=Lx, s_b=Ly * Lx, nbi=nz)
        d.out = H.Lines.make([x1.data_ptr()], Kx, **self._et(T, Ly * T, T), s_b=Kx * Ly, nbi=nz)
        self.ctx.hd_pass(self.dt, d)
        d = self._desc(H.HD_PASS_FWD, 1, Kx, nz, T)
        d.in_f = H.Lines.make([x1.data_ptr()], Ly, **self._lt(T, Ly * T), s_j=T, s_b=Kx * Ly, nbi=nz)
        d.out = H.Lines.make([out_ptr], self.ax[1]["M1"], **self._lt(T, s_t), s_j=s_ky, jd=jd, s_jt=s_jt,
                             s_b=s_z, nbi=nz)
        d.batch_fastest = 1
        self.ctx.hd_pass(self.dt, d)

    def fwd_planes(self, f_planes, nz, send, P):
        if nz <= 0:
            return
        # element (zl, ky, kx) -> P.ex1(ky / Kys, ky % Kys, kx, zl)
        tiled = P.Kys < P.Ky
        self._xy(f_planes, nz, P.Lf[1], P.Lf[2], send.data_ptr(), s_ky=P.Kx * P.Rz, s_t=P.Rz * P.T, s_z=P.T,
                 T=P.T, jd=P.Kys if tiled else 0, s_jt=P.block1 if tiled else 0)

    def fwd_g(self, g, xyg, P):
        # XYg[ky][kx/T][z][kx%T]
        self._xy(g, P.Lg[0], P.Lg[1], P.Lg[2], xyg.data_ptr(), s_ky=P.Kx * P.Lg[0], s_t=P.Lg[0] * P.T,
                 s_z=P.T, T=P.T)

    def conv_lines(self, recv1, xyg, ky0, nky, send2, P):
        if nky <= 0:
            return
        H, T = self.H, P.T
        eb = xyg.element_size()
        d = self._desc(H.HD_PASS_CONV, 0, P.Kx, nky, T)
        # element z = src * Rz + zl of line kx, batch kyl: P.ex1(src, kyl, kx, zl)
        d.in_f = H.Lines.make([recv1.data_ptr()], P.Lf[0], **self._lt(T, P.Rz * T), s_j=T,
                              jd=P.Rz if P.Rz < P.Lf[0] else 0, s_jt=P.block1, s_b=P.Kx * P.Rz, nbi=nky)
        d.in_g = H.Lines.make([xyg.data_ptr() + ky0 * P.Kx * P.Lg[0] * eb], P.Lg[0], **self._lt(T, P.Lg[0] * T), s_j=T, s_b=P.Kx * P.Lg[0], nbi=nky)
        # element zo = dst * Roz + zol: P.ex2(dst, zol, kx, kyl)
        d.out = H.Lines.make([send2.data_ptr()], P.O[0], **self._lt(T, P.Kys * T), s_j=P.Kx * P.Kys,
                             jd=P.Roz if P.Roz < P.O[0] else 0, s_jt=P.block2, s_b=T, nbi=nky)
        d.scale = self.scale
        d.batch_fastest = 1
        self.ctx.hd_pass(self.dt, d)

    def inv_planes(self, recv2, nzo, P):
        h = self.torch.empty((max(nzo, 0), P.O[1], P.O[2]), dtype=self.tdt, device=self.dev)
        if nzo <= 0:
            return h
        H, T = self.H, P.T
        Oyp = -(-P.O[1] // T) * T
        w = self.empty(nzo * Oyp * P.Kx)                               # W[zol][y/T][kx][y%T]
        d = self._desc(H.HD_PASS_INV, 1, P.Kx, nzo, T)
        # element ky = src * Kys + kyl of line kx, batch zol: P.ex2(src, zol, kx, kyl)
        d.in_f = H.Lines.make([recv2.data_ptr()], P.Ky, **self._lt(T, P.Kys * T), s_j=T,
                              jd=P.Kys if P.Kys < P.Ky else 0, s_jt=P.block2, s_b=P.Kx * P.Kys, nbi=nzo)
        d.out = H.Lines.make([w.data_ptr()], P.O[1], **self._et(T, P.Kx * T, T), s_b=Oyp * P.Kx, nbi=nzo)
        self.ctx.hd_pass(self.dt, d)
        d = self._desc(H.HD_PASS_INV, 2, P.O[1], nzo, T)
        d.in_f = H.Lines.make([w.data_ptr()], P.Kx, **self._lt(T, P.Kx * T), s_j=T, s_b=Oyp * P.Kx, nbi=nzo)
        d.out = H.Lines.make([h.data_ptr()], P.O[2], s_l=P.O[2], s_b=P.O[1] * P.O[2], nbi=nzo)
        self.ctx.hd_pass(self.dt, d)
        return h


def torch_exchange(group=None):
    """all-to-all of equal contiguous blocks with torch.distributed (NCCL on GPU)."""
    import torch.distributed as dist

    def ex(send, recv, block):
        n = dist.get_world_size(group)
        dist.all_to_all_single(recv[: n * block], send[: n * block], group=group)
    return ex
