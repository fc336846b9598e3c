"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no transforms, no twiddles,
no convolution).  It only draws numbers.  Both sides of every parity test get
their inputs from here, so the oracle and the CUDA path never feed each other.

Generator (SURVEY.md §8(d) generator rules):
  * counter-based splitmix64: draw i of a stream with seed S is
    mix64(S + (i + 1) * 0x9E3779B97F4A7C15)  (the splitmix64 finaliser),
  * u = (x >> 11) * 2**-53  in [0, 1),
  * arrays are drawn in the order the recipe lists them, row-major,
    re then im per complex sample, each array continuing the stream counter,
  * complex64 inputs are drawn in double and then rounded.

The BASELINE.json configs (configs[0..4]) are reproduced by `config_inputs`.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class Stream:
    """One splitmix64 stream; `uniform(n)` returns the next n draws in [0,1)."""

    def __init__(self, seed: int = 0):
        self.seed = np.uint64(seed)
        self.counter = 0

    def uniform(self, n: int, chunk: int = 1 << 24) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        with np.errstate(over="ignore"):
            for lo in range(0, n, chunk):
                hi = min(n, lo + chunk)
                i = np.arange(self.counter + lo + 1, self.counter + hi + 1, dtype=np.uint64)
                x = _mix64(self.seed + i * GOLDEN)
                out[lo:hi] = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        self.counter += n
        return out

    def complex_uniform(self, shape, lo=-1.0, hi=1.0, dtype=np.complex128) -> np.ndarray:
        n = int(np.prod(shape))
        u = self.uniform(2 * n)
        v = lo + (hi - lo) * u
        z = (v[0::2] + 1j * v[1::2]).reshape(shape)
        return z.astype(dtype)

    def real_uniform(self, shape, lo=0.0, hi=1.0) -> np.ndarray:
        n = int(np.prod(shape))
        return (lo + (hi - lo) * self.uniform(n)).reshape(shape)


def random_pair(seed, shape_f, shape_g, dtype=np.complex128, lo=-1.0, hi=1.0):
    """f then g from one stream (used by the randomised small-problem sweeps)."""
    s = Stream(seed)
    f = s.complex_uniform(shape_f, lo, hi, dtype)
    g = s.complex_uniform(shape_g, lo, hi, dtype)
    return f, g


def integer_pair(seed, shape_f, shape_g, lim=8):
    """Complex inputs with integer re/im in [-lim, lim] (exactness pins, O6)."""
    s = Stream(seed)
    def draw(shape):
        n = int(np.prod(shape))
        u = s.uniform(2 * n)
        v = np.floor(u * (2 * lim + 1)) - lim
        return (v[0::2] + 1j * v[1::2]).reshape(shape)
    return draw(shape_f), draw(shape_g)


# --------------------------------------------------------------------------
# BASELINE.json configs.  Each returns dict(ndim, dtype, f=[...], g=[...], plan)
# --------------------------------------------------------------------------
CONFIG_NAMES = {
    1: "1d_c128_64x40",
    2: "1d_c128_batch4096_8192x3000",
    3: "2d_c128_4096sq_x_255sq_gauss",
    4: "3d_c64_512cube_x_129cube",
    5: "2d_c128_multiconv6_2048sq_x_1024x1536",
}


def gaussian_kernel(stream: Stream, n=255, sigma=40.0, noise=1e-3):
    """Config 3 kernel: exp(-((a-c)^2+(b-c)^2)/(2 sigma^2)) + noise*u, real."""
    c = (n - 1) / 2.0
    a = np.arange(n, dtype=np.float64) - c
    base = np.exp(-(a[:, None] ** 2 + a[None, :] ** 2) / (2.0 * sigma * sigma))
    return (base + noise * stream.real_uniform((n, n))).astype(np.complex128)


def config_inputs(cfg: int, batch: int | None = None, scale: int = 1):
    """Inputs of BASELINE.json configs[cfg-1] (seed 0, one stream per config).

    `batch` truncates config 2's pair count (the stream order is unchanged:
    all f rows are drawn before g, so a truncated batch uses the first rows of
    each array as drawn for the full config only when batch == 4096; smaller
    batches are their own seeded stream, documented as such).
    `scale` divides the spatial extents (used by reduced parity cases).
    """
    s = Stream(0)
    if cfg == 1:
        f = s.complex_uniform((64,))
        g = s.complex_uniform((40,))
        return dict(ndim=1, batch=1, dtype="c128", f=[f], g=[g], M=None,
                    plan=dict(m=32, q=4))
    if cfg == 2:
        B = 4096 if batch is None else batch
        f = s.complex_uniform((B, 8192 // scale))
        g = s.complex_uniform((B, 3000 // scale))
        return dict(ndim=1, batch=B, dtype="c128", f=[f], g=[g], M=None, plan=None)
    if cfg == 3:
        n = 4096 // scale
        k = 255 if scale == 1 else max(3, (255 // scale) | 1)
        img = s.real_uniform((n, n)).astype(np.complex128)
        ker = gaussian_kernel(s, k, 40.0 / scale)
        return dict(ndim=2, batch=1, dtype="c128", f=[img], g=[ker], M=None, plan=None)
    if cfg == 4:
        n, k = 512 // scale, max(3, 129 // scale)
        f = s.complex_uniform((n, n, n), dtype=np.complex128).astype(np.complex64)
        g = s.complex_uniform((k, k, k), dtype=np.complex128).astype(np.complex64)
        return dict(ndim=3, batch=1, dtype="c64", f=[f], g=[g], M=None, plan=None)
    if cfg == 5:
        fs, gs = [], []
        for _ in range(6):
            fs.append(s.complex_uniform((2048 // scale, 2048 // scale)))
            gs.append(s.complex_uniform((1024 // scale, 1536 // scale)))
        return dict(ndim=2, batch=1, dtype="c128", f=fs, g=gs, M=None, plan=None)
    raise ValueError(cfg)


def sample_indices(out_shape, n_random=4096, seed=12345, edge=8):
    """Seeded output-index sample for full-size parity: every corner, the first and
    last `edge` indices along each axis (others at random), plus n_random uniform
    random indices.  Returns int64 array [n, ndim] (duplicates removed)."""
    out_shape = [int(v) for v in out_shape]
    nd = len(out_shape)
    s = Stream(seed)
    rows = []
    # corners
    for c in range(1 << nd):
        rows.append([(out_shape[i] - 1) if (c >> i) & 1 else 0 for i in range(nd)])
    # edges along each axis
    for ax in range(nd):
        for e in list(range(min(edge, out_shape[ax]))) + \
                list(range(max(0, out_shape[ax] - edge), out_shape[ax])):
            u = s.uniform(nd)
            r = [int(u[i] * out_shape[i]) for i in range(nd)]
            r[ax] = e
            rows.append(r)
    u = s.uniform(n_random * nd).reshape(n_random, nd)
    rnd = np.floor(u * np.asarray(out_shape, dtype=np.float64)).astype(np.int64)
    idx = np.concatenate([np.asarray(rows, dtype=np.int64).reshape(-1, nd), rnd])
    return np.unique(idx, axis=0)


def unit_torus_points(npts, ndim, seed=777):
    """Random points on the unit torus |z_i| = 1 (polynomial-identity checks)."""
    s = Stream(seed)
    u = s.uniform(npts * ndim).reshape(npts, ndim)
    return np.exp(2j * np.pi * u)
