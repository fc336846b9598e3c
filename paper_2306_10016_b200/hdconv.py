"""Thin ctypes binding of libhdconv.so (include/hdconv.h).

Argument marshalling only: every step of the convolution runs in the CUDA
kernels of libhdconv.so.  There is no CPU fallback: importing this module
without the built library raises, and every compute call on a machine without
a CUDA device raises HDError(HD_ERR_CUDA).

Tensors are torch tensors on the context's device (complex128 -> HD_C128,
complex64 -> HD_C64), row-major and contiguous.  The function names mirror the
C entry points (hd_conv1d, hd_conv2d, ...).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhdconv.so")

HD_C64, HD_C128 = 1, 2
HD_OK, HD_ERR_INVALID, HD_ERR_UNSUPPORTED, HD_ERR_CUDA, HD_ERR_NCCL, HD_ERR_WORKSPACE = range(6)
HD_FLAG_ALLOW_ALIAS = 0x1
HD_FLAG_SHARED_G = 0x2
HD_FLAG_GENERIC_FFT = 0x4
HD_FLAG_GRAPH = 0x8
HD_FLAG_STAGED_ORDER = 0x10
HD_FLAG_EXPLICIT_PLAN = 0x20
HD_ENGINE_GENERIC, HD_ENGINE_S512, HD_ENGINE_S512_MCONV, HD_ENGINE_S128, HD_ENGINE_S512C, HD_ENGINE_S2048R, \
    HD_ENGINE_S4096R = range(7)
HD_TUNE_PER_AXIS = 0x0
HD_TUNE_EXHAUSTIVE = 0x1
HD_MAX_DIM = 3
HD_MAX_PAIRS = 16

STATUS_NAMES = {0: "HD_OK", 1: "HD_ERR_INVALID", 2: "HD_ERR_UNSUPPORTED", 3: "HD_ERR_CUDA",
                4: "HD_ERR_NCCL", 5: "HD_ERR_WORKSPACE"}

EXPORTED = [
    "hd_abi_version", "hd_create", "hd_destroy", "hd_last_error", "hd_plan_default",
    "hd_plan_complete", "hd_spectral_permutation", "hd_workspace_bytes", "hd_conv1d",
    "hd_conv2d", "hd_conv3d", "hd_multiconv", "hd_conv_explicit", "hd_conv_host", "hd_conv_window",
    "hd_conv_real",
    "hd_conv_host_async", "hd_host_sync",
    "hd_forward_residues", "hd_backward_residues", "hd_tune", "hd_tune_ex", "hd_tune_log",
    "hd_profile_enable", "hd_profile_read", "hd_profile_reset", "hd_launch_count", "hd_engine_launches", "hd_graph_replays", "hd_pass", "hd_conv1d_lambda",
    "hd_dist_unique_id", "hd_dist_init", "hd_dist_last_error", "hd_dist_partition", "hd_dist_slab_plan",
    "hd_conv1d_dist", "hd_conv2d_dist", "hd_conv3d_dist", "hd_slab_stage", "hd_slab_scratch_bytes",
    "hd_slab_g_bytes", "hd_tune_explicit", "hd_tune_space", "hd_filter_kernel", "hd_filter_image", "hd_filter_last_error",
]
HD_FILTER_COUNT = 8
FILTER_NAMES = ["Identity", "Ridge_detection_1", "Ridge_detection_2", "Sharpen", "Box_blur", "Gaussian_blur",
                "Gaussian_blur_5", "Unsharpen_masking"]
HD_SHARD_BATCH, HD_SHARD_RESIDUE = 0, 1
HD_PASS_FWD, HD_PASS_INV, HD_PASS_CONV = 0, 1, 2


class AxisPlan(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("p_f", ctypes.c_int32), ("p_g", ctypes.c_int32),
                ("q", ctypes.c_int32), ("C", ctypes.c_int32), ("S", ctypes.c_int32),
                ("D", ctypes.c_int32), ("threads", ctypes.c_int32), ("M1", ctypes.c_int64)]


class Plan(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("axis", AxisPlan * HD_MAX_DIM), ("tuned_seconds", ctypes.c_double)]

    def as_dict(self):
        return {"ndim": self.ndim, "flags": self.flags, "tuned_seconds": self.tuned_seconds,
                "axis": [{f: getattr(self.axis[i], f) for f, _ in AxisPlan._fields_}
                         for i in range(self.ndim)]}

    @staticmethod
    def make(ndim, axes, flags=0):
        """axes: list of dicts with m and optional C, S, D (0 = default)."""
        p = Plan()
        p.ndim = ndim
        p.flags = flags
        for i, a in enumerate(axes):
            p.axis[i].m = int(a["m"])
            p.axis[i].C = int(a.get("C", 0))
            p.axis[i].S = int(a.get("S", 0))
            p.axis[i].D = int(a.get("D", 0))
            p.axis[i].threads = int(a.get("threads", 0))
        return p


HD_TUNE_RANDOM = 0x2


class TuneOpts(ctypes.Structure):
    """hd_tune_opts_t (include/hdconv.h)."""
    _fields_ = [("flags", ctypes.c_uint32), ("reps", ctypes.c_int32), ("n1", ctypes.c_int32),
                ("fake_cost", ctypes.c_int32), ("seed", ctypes.c_uint64), ("proxy_rows", ctypes.c_int64)]


class Lines(ctypes.Structure):
    """hd_lines_t: element j of line l, batch b, array k at
    ptr[k] + (b/nbi)*s_bo + (b%nbi)*s_b + line(l) + elem(j) (see include/hdconv.h)."""
    _fields_ = [("ptr", ctypes.c_void_p * HD_MAX_PAIRS), ("L", ctypes.c_int64),
                ("nbi", ctypes.c_int64), ("s_bo", ctypes.c_int64), ("s_b", ctypes.c_int64),
                ("tl", ctypes.c_int32), ("pad_", ctypes.c_int32), ("s_t", ctypes.c_int64),
                ("s_l", ctypes.c_int64), ("jd", ctypes.c_int64), ("s_jt", ctypes.c_int64),
                ("s_j", ctypes.c_int64)]

    @staticmethod
    def make(ptrs, L, s_l, s_j=1, jd=0, s_jt=0, s_b=0, nbi=0, s_bo=0, tl=40, s_t=0):
        d = Lines()
        for k, q in enumerate(ptrs):
            d.ptr[k] = q
        d.L, d.s_l, d.s_j, d.jd, d.s_jt = L, s_l, s_j, jd, s_jt
        d.s_b, d.nbi, d.s_bo, d.tl, d.s_t = s_b, nbi, s_bo, tl, s_t
        return d


class PassDesc(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("npairs", ctypes.c_int32), ("nlines", ctypes.c_int64),
                ("nbatch", ctypes.c_int64), ("M", ctypes.c_int64), ("axis", AxisPlan),
                ("in_f", Lines), ("in_g", Lines), ("out", Lines), ("scale", ctypes.c_double),
                ("batch_fastest", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("r_begin", ctypes.c_int32), ("r_end", ctypes.c_int32)]


class SlabPlan(ctypes.Structure):
    """hd_slab_plan_t: one rank's share of a 2-D / 3-D slab decomposition (include/hdconv.h)."""
    _fields_ = [("ndim", ctypes.c_int32), ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nchunks", ctypes.c_int32),
                ("in_lo", ctypes.c_int64), ("in_hi", ctypes.c_int64), ("out_lo", ctypes.c_int64),
                ("out_hi", ctypes.c_int64), ("spec_lo", ctypes.c_int64), ("spec_hi", ctypes.c_int64),
                ("R", ctypes.c_int64), ("Ro", ctypes.c_int64), ("Ks", ctypes.c_int64),
                ("chunk_rows", ctypes.c_int64), ("chunk_cols", ctypes.c_int64),
                ("block1", ctypes.c_int64), ("block2", ctypes.c_int64), ("bytes_sent", ctypes.c_int64),
                ("scale", ctypes.c_double), ("plan", Plan)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "plan"}
        d["plan"] = self.plan.as_dict()
        return d


class HDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2306_10016_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
    PP = ctypes.POINTER(Plan)
    sig = {
        "hd_abi_version": ([], ctypes.c_int),
        "hd_create": ([ctypes.POINTER(P), ctypes.c_int], ctypes.c_int),
        "hd_destroy": ([P], ctypes.c_int),
        "hd_last_error": ([P], ctypes.c_char_p),
        "hd_plan_default": ([ctypes.c_int, I32, I32, P, P, P, PP], ctypes.c_int),
        "hd_plan_complete": ([ctypes.c_int, I32, I32, P, P, P, PP], ctypes.c_int),
        "hd_spectral_permutation": ([I32, P], ctypes.c_int),
        "hd_workspace_bytes": ([P, ctypes.c_int, I32, I32, I64, P, P, P, PP], SZ),
        "hd_conv1d": ([P, ctypes.c_int, I64, P, I64, P, I64, P, I64, PP, P, SZ, P], ctypes.c_int),
        "hd_conv2d": ([P, ctypes.c_int, I64, P, P, P, P, P, P, PP, P, SZ, P], ctypes.c_int),
        "hd_conv3d": ([P, ctypes.c_int, I64, P, P, P, P, P, P, PP, P, SZ, P], ctypes.c_int),
        "hd_multiconv": ([P, ctypes.c_int, I32, I32, P, P, P, P, P, P, PP, P, SZ, P], ctypes.c_int),
        "hd_conv_explicit": ([P, ctypes.c_int, I32, I32, P, P, P, P, P, PP, P], ctypes.c_int),
        "hd_conv_real": ([P, ctypes.c_int, I32, I64, P, P, P, P, P, PP, P], ctypes.c_int),
        "hd_conv_window": ([P, ctypes.c_int, I32, I32, I64, P, P, P, P, P, P, P, P, PP, P, ctypes.c_size_t, P],
                           ctypes.c_int),
        "hd_conv_host": ([P, ctypes.c_int, I32, I32, I64, P, P, P, P, P, P, PP, P], ctypes.c_int),
        "hd_conv_host_async": ([P, ctypes.c_int, I32, I32, I64, P, P, P, P, P, P, PP], ctypes.c_int),
        "hd_host_sync": ([P], ctypes.c_int),
        "hd_forward_residues": ([P, ctypes.c_int, I64, P, I64, I32, I32, P, P], ctypes.c_int),
        "hd_backward_residues": ([P, ctypes.c_int, I64, P, I32, I32, P, I64, P], ctypes.c_int),
        "hd_tune": ([P, ctypes.c_int, I32, I32, I64, P, P, P, U32, I32, P, PP], ctypes.c_int),
        "hd_tune_ex": ([P, ctypes.c_int, I32, I32, I64, P, P, P, ctypes.POINTER(TuneOpts), P, PP], ctypes.c_int),
        "hd_tune_log": ([P, I32, PP, P], I32),
        "hd_profile_enable": ([P, I32], ctypes.c_int),
        "hd_profile_read": ([P, I32, P, P, P], I32),
        "hd_profile_reset": ([P], ctypes.c_int),
        "hd_launch_count": ([P], I64),
        "hd_engine_launches": ([P, I32], I64),
        "hd_graph_replays": ([P], I64),
        "hd_conv1d_lambda": ([P, ctypes.c_int, I64, P, I64, P, I64, P, I64, I32, I32, P], ctypes.c_int),
        "hd_pass": ([P, ctypes.c_int, ctypes.POINTER(PassDesc), P], ctypes.c_int),
        "hd_dist_unique_id": ([P], ctypes.c_int),
        "hd_dist_init": ([P, P, I32, I32], ctypes.c_int),
        "hd_dist_last_error": ([], ctypes.c_char_p),
        "hd_dist_partition": ([I64, I32, I32, P, P], ctypes.c_int),
        "hd_dist_slab_plan": ([ctypes.c_int, I32, I32, I32, I32, P, P, PP, ctypes.POINTER(SlabPlan)],
                              ctypes.c_int),
        "hd_conv1d_dist": ([P, ctypes.c_int, I64, P, I64, P, I64, P, PP, U32, P], ctypes.c_int),
        "hd_conv2d_dist": ([P, ctypes.c_int, P, P, P, P, P, PP, I32, P], ctypes.c_int),
        "hd_conv3d_dist": ([P, ctypes.c_int, P, P, P, P, P, PP, P], ctypes.c_int),
        "hd_slab_stage": ([P, ctypes.c_int, ctypes.POINTER(SlabPlan), P, P, I32, P, P, P, P, P], ctypes.c_int),
        "hd_slab_scratch_bytes": ([ctypes.c_int, ctypes.POINTER(SlabPlan), P, P], SZ),
        "hd_slab_g_bytes": ([ctypes.c_int, ctypes.POINTER(SlabPlan), P], SZ),
        "hd_filter_kernel": ([I32, P, ctypes.POINTER(I32), ctypes.POINTER(ctypes.c_char_p)], ctypes.c_int),
        "hd_tune_explicit": ([P, ctypes.c_int, I32, I32, P, P, I32, P, PP], ctypes.c_int),
        "hd_tune_space": ([ctypes.c_int, I32, I32, P, P, P, I32, ctypes.POINTER(AxisPlan), I32], I32),
        "hd_filter_image": ([P, ctypes.c_int, P, I64, I64, I32, I32, I32, P, P, P, P], ctypes.c_int),
        "hd_filter_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = _load()


def lib():
    return _lib


def _i64arr(v):
    a = (ctypes.c_int64 * len(v))(*[int(x) for x in v])
    return a


def _check(status, ctx=None):
    if status != HD_OK:
        msg = _lib.hd_last_error(ctx)
        raise HDError(status, msg.decode() if msg else "")


def _check_dist(status, ctx=None):
    """Status of a distributed entry point: its own message, else the pass's."""
    if status != HD_OK:
        msg = _lib.hd_dist_last_error() or b""
        if not msg and ctx is not None:
            msg = _lib.hd_last_error(ctx) or b""
        raise HDError(status, msg.decode())


def dist_partition(extent, nranks, rank):
    """[lo, hi) of `extent` items owned by `rank` (hd_dist_partition)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check_dist(_lib.hd_dist_partition(int(extent), int(nranks), int(rank), ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def tune_space(dtype, Lf, Lg, axis, M=None, N=1):
    """hd_tune_space: the per-axis candidates of hd_tune as (m, C, S, D, threads) tuples."""
    Mv = _i64arr(M) if M is not None else None
    n = _lib.hd_tune_space(dtype, len(Lf), N, _i64arr(Lf), _i64arr(Lg), Mv, axis, None, 0)
    if n < 0:
        raise HDError(HD_ERR_INVALID, "bad tune_space arguments")
    arr = (AxisPlan * max(n, 1))()
    _lib.hd_tune_space(dtype, len(Lf), N, _i64arr(Lf), _i64arr(Lg), Mv, axis, arr, n)
    return [(a.m, a.C, a.S, a.D, a.threads) for a in arr[:n]]


def filter_kernel(kernel):
    """(name, n x n weights) of the paper's filter dictionary entry (id or name)."""
    kid = FILTER_NAMES.index(kernel) if isinstance(kernel, str) else int(kernel)
    w = np.zeros(25, dtype=np.float64)
    n, name = ctypes.c_int32(), ctypes.c_char_p()
    st = _lib.hd_filter_kernel(kid, w.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n), ctypes.byref(name))
    if st != HD_OK:
        raise HDError(st, (_lib.hd_filter_last_error() or b"").decode())
    return name.value.decode(), w[: n.value * n.value].reshape(n.value, n.value)


def slab_buffer_elems(dtype, sp, Lf, Lg):
    """Element counts of a rank's slab buffers: transformed g, send/recv 1 and 2, 3-D scratch."""
    esz = 16 if dtype == HD_C128 else 8
    g = _lib.hd_slab_g_bytes(dtype, ctypes.byref(sp), _i64arr(Lg)) // esz
    sc = _lib.hd_slab_scratch_bytes(dtype, ctypes.byref(sp), _i64arr(Lf), _i64arr(Lg)) // esz
    return dict(g=int(g), x1=int(sp.nranks * sp.block1), x2=int(sp.nranks * sp.block2), scratch=int(sc))


def slab_plan(dtype, Lf, Lg, nranks, rank, nchunks=0, plan=None):
    """hd_dist_slab_plan (host only): this rank's rows/planes, spectral lines, exchange blocks."""
    sp = SlabPlan()
    pp = ctypes.byref(plan) if plan is not None else None
    _check_dist(_lib.hd_dist_slab_plan(dtype, len(Lf), int(nranks), int(rank), int(nchunks), _i64arr(Lf),
                                       _i64arr(Lg), pp, ctypes.byref(sp)))
    return sp


def _dtype_code(t):
    import torch
    if t.dtype == torch.complex128:
        return HD_C128
    if t.dtype == torch.complex64:
        return HD_C64
    raise TypeError(f"unsupported dtype {t.dtype} (complex64 / complex128 only)")


def _stream_ptr(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):  # torch.cuda.Stream
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))  # a raw cudaStream_t


def _ptr(t):
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------
# host-only helpers (no GPU required)
# ---------------------------------------------------------------------------
def hd_plan_default(dtype, Lf, Lg, M=None, npairs=1):
    ndim = len(Lf)
    p = Plan()
    Mv = _i64arr(M) if M is not None else None
    _check(_lib.hd_plan_default(dtype, ndim, npairs, _i64arr(Lf), _i64arr(Lg), Mv, ctypes.byref(p)))
    return p


def hd_plan_complete(dtype, Lf, Lg, plan, M=None, npairs=1):
    Mv = _i64arr(M) if M is not None else None
    _check(_lib.hd_plan_complete(dtype, len(Lf), npairs, _i64arr(Lf), _i64arr(Lg), Mv,
                                 ctypes.byref(plan)))
    return plan


def hd_spectral_permutation(m):
    perm = np.zeros(m, dtype=np.int32)
    _check(_lib.hd_spectral_permutation(m, perm.ctypes.data_as(ctypes.c_void_p)))
    return perm


def hd_abi_version():
    return _lib.hd_abi_version()


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------
# ---------------------------------------------------------------------------
# Tuning-record analysis of the paper's heuristics (host logic, no device work)
def sort_lists_topk(A, B, k):
    """Pairs (A_i, B_i) sorted ascending by B (stable); the first k of each and their
    original indices (the appendix optimisation code's sort-and-take-k helper)."""
    if len(A) != len(B):
        raise ValueError("length mismatch")
    idx = sorted(range(len(B)), key=lambda i: B[i])[:max(0, k)]
    return [A[i] for i in idx], [B[i] for i in idx], idx


def sort_lists_eps(A, B, eps):
    """Algorithm 'Sort lists by threshold': with t_best = min B,
    t_worst = max B and T = t_best + eps (t_worst - t_best), the a_i with b_i <= T,
    ascending in b, paired with (b_i - t_best) / (t_worst - t_best) (0 when all equal)."""
    if len(A) != len(B) or not A:
        raise ValueError("need equal, non-empty lists")
    tb, tw = min(B), max(B)
    T = tb + eps * (tw - tb)
    out_a, out_b = [], []
    for i in sorted(range(len(B)), key=lambda i: B[i]):
        if B[i] <= T:
            out_a.append(A[i])
            out_b.append(0.0 if tw == tb else (B[i] - tb) / (tw - tb))
    return out_a, out_b


def epsilon_smallest_rectangle(square, rects, eps):
    """Smallest rectangle height whose eps-filtered m list contains the square's best
    m (the algorithm's gamma = t_best + eps (t_worst - t_best)).
    square = (m_values, times); rects = {L_y: (m_values, times)}; None if none does."""
    ms, ts = square
    if not ms:
        raise ValueError("empty square record")
    m_star = ms[min(range(len(ts)), key=lambda i: ts[i])]
    for ly in sorted(rects):
        a, b = rects[ly]
        if m_star in sort_lists_eps(list(a), list(b), eps)[0]:
            return ly
    return None


def skinny_estimate(square, rect):
    """The L_y = 32 heuristic: the rectangle's best m, the square's
    time at that m, and the square's own optimum; transfer miss if the square never
    timed that m.  Returns (m_transfer, time_at_transfer, m_best, time_best) or
    ('miss', m_transfer, m_best, time_best)."""
    (ms, ts), (mr, tr) = square, rect
    if not ms or not mr:
        raise ValueError("empty record")
    m_t = mr[min(range(len(tr)), key=lambda i: tr[i])]
    ib = min(range(len(ts)), key=lambda i: ts[i])
    if m_t not in ms:
        return ("miss", m_t, ms[ib], ts[ib])
    return (m_t, ts[ms.index(m_t)], ms[ib], ts[ib])


def window_for_mode(mode, Lf, Lg):
    """(lo, n) per axis for the output modes of the paper's 2-D listing
    (N = L1 + L2 - 1 with L1 = L_f, L2 = L_g as in its call
    mainconvolve(f, g, ...)): full [0, N); same_big [0, L2); same_small [1, 1 + L1);
    valid [ceil(N/L2) - 1, ceil(N/L1) + 1) -- the listing's formula as written
    (SPEC.md flags it as differing from the conventional valid size), clipped to
    the output."""
    lo, n = [], []
    for a, b in zip(Lf, Lg):
        N = a + b - 1
        if mode == "full":
            v, v1 = 0, N
        elif mode == "same_big":
            v, v1 = 0, b
        elif mode == "same_small":
            v, v1 = 1, 1 + a
        elif mode == "valid":
            v, v1 = -(-N // b) - 1, -(-N // a) + 1
        else:
            raise ValueError(f"unknown mode {mode!r}: full, same_big, same_small, valid")
        v, v1 = max(0, v), min(N, v1)
        if v1 <= v:
            raise ValueError(f"empty {mode} window for extents {a}, {b}")
        lo.append(v)
        n.append(v1 - v)
    return lo, n


class Context:
    """One hd_ctx_t bound to a CUDA device (owns twiddle tables, plan cache, scratch)."""

    def __init__(self, device=0):
        h = ctypes.c_void_p()
        _check(_lib.hd_create(ctypes.byref(h), int(device)))
        self.h = h
        self.device = device
        self.world, self.rank = 1, 0

    def close(self):
        if self.h:
            _lib.hd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        _check(st, self.h)

    # ---- convolution (device tensors) --------------------------------------
    def _out(self, like, shape):
        import torch
        return torch.empty(shape, dtype=like.dtype, device=like.device)

    def _arg(self, t, name, dtype, shape=None):
        """Validate a device tensor before its pointer crosses the ABI: the kernels
        trust dtype, extents, contiguity and device."""
        if not hasattr(t, "data_ptr") or not hasattr(t, "device"):
            raise TypeError(f"{name} must be a torch tensor")
        if t.device.type != "cuda" or (t.device.index or 0) != int(self.device):
            raise ValueError(f"{name} is on {t.device}, the context is on cuda:{self.device}")
        if t.dtype != dtype:
            raise TypeError(f"{name} has dtype {t.dtype}, expected {dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if shape is not None and list(t.shape) != [int(v) for v in shape]:
            raise ValueError(f"{name} has shape {list(t.shape)}, expected {[int(v) for v in shape]}")
        return t

    def _pairs(self, fs, gs, batch=False, shared_g=False):
        """Validate the operand lists of a (multi-)convolution: every f_k shares f_0's
        dtype and shape, every g_k g_0's; the batch axis of g is 1 or absent only with
        shared_g."""
        if len(fs) != len(gs) or not fs:
            raise ValueError("need the same number (>= 1) of f and g arrays")
        f0, g0 = fs[0], gs[0]
        _dtype_code(f0)
        nd = f0.dim() - (1 if batch else 0)
        if not 1 <= nd <= 3:
            raise ValueError("ndim must be 1, 2 or 3")
        for k, f in enumerate(fs):
            self._arg(f, f"f[{k}]", f0.dtype, f0.shape)
        if batch and not shared_g:
            gshape = [f0.shape[0]] + list(g0.shape[-nd:])
        elif batch and g0.dim() == nd + 1:
            gshape = [1] + list(g0.shape[-nd:])
        else:
            gshape = list(g0.shape[-nd:])
        if g0.dim() not in (nd, nd + 1) or (g0.dim() == nd + 1 and not batch):
            raise ValueError(f"g has {g0.dim()} dims, expected {nd}" + (" (+ batch)" if batch else ""))
        for k, g in enumerate(gs):
            self._arg(g, f"g[{k}]", f0.dtype, gshape)
        return nd

    def _h(self, h, like, shape):
        if h is None:
            return self._out(like, shape)
        return self._arg(h, "h", like.dtype, shape)

    def conv(self, f, g, M=None, plan=None, h=None, batch=False, shared_g=False, stream=None):
        """Full linear convolution of torch tensors f, g (1-3 dims, leading batch
        axis when batch=True)."""
        nd = self._pairs([f], [g], batch, shared_g)
        B = f.shape[0] if batch else 1
        Lf = list(f.shape[-nd:])
        Lg = list(g.shape[-nd:])
        if plan is None and shared_g:
            plan = self.default_plan(_dtype_code(f), Lf, Lg, M)
        if plan is not None:
            plan = Plan.from_buffer_copy(plan)  # never mutate the caller's plan
            if shared_g:
                plan.flags |= HD_FLAG_SHARED_G
            else:
                plan.flags &= ~HD_FLAG_SHARED_G
        out_shape = ([B] if batch else []) + [a + b - 1 for a, b in zip(Lf, Lg)]
        if plan is not None and (plan.flags & HD_FLAG_ALLOW_ALIAS):
            pc = hd_plan_complete(_dtype_code(f), Lf, Lg, Plan.from_buffer_copy(plan), M)
            out_shape = ([B] if batch else []) + [min(a + b - 1, pc.axis[i].M1)
                                                  for i, (a, b) in enumerate(zip(Lf, Lg))]
        h = self._h(h, f, out_shape)
        dt = _dtype_code(f)
        Mv = _i64arr(M) if M is not None else _i64arr([0] * nd)
        pp = ctypes.byref(plan) if plan is not None else None
        st = _stream_ptr(stream)
        if nd == 1:
            self._chk(_lib.hd_conv1d(self.h, dt, B, _ptr(f), Lf[0], _ptr(g), Lg[0], _ptr(h),
                                     int(M[0]) if M is not None else 0, pp, None, 0, st))
        elif nd == 2:
            self._chk(_lib.hd_conv2d(self.h, dt, B, _ptr(f), _i64arr(Lf), _ptr(g), _i64arr(Lg),
                                     _ptr(h), Mv, pp, None, 0, st))
        elif nd == 3:
            self._chk(_lib.hd_conv3d(self.h, dt, B, _ptr(f), _i64arr(Lf), _ptr(g), _i64arr(Lg),
                                     _ptr(h), Mv, pp, None, 0, st))
        else:
            raise ValueError("ndim must be 1, 2 or 3")
        return h

    def hd_conv1d(self, f, g, **kw):
        return self.conv(f, g, **kw)

    def hd_conv2d(self, f, g, **kw):
        return self.conv(f, g, **kw)

    def hd_conv3d(self, f, g, **kw):
        return self.conv(f, g, **kw)

    def hd_multiconv(self, fs, gs, M=None, plan=None, h=None, stream=None):
        """h = sum_k fs[k] * gs[k]."""
        N = len(fs)
        nd = self._pairs(fs, gs)
        Lf, Lg = list(fs[0].shape), list(gs[0].shape)
        h = self._h(h, fs[0], [a + b - 1 for a, b in zip(Lf, Lg)])
        fp = (ctypes.c_void_p * N)(*[t.data_ptr() for t in fs])
        gp = (ctypes.c_void_p * N)(*[t.data_ptr() for t in gs])
        Mv = _i64arr(M) if M is not None else None
        pp = ctypes.byref(plan) if plan is not None else None
        self._chk(_lib.hd_multiconv(self.h, _dtype_code(fs[0]), nd, N, fp, _i64arr(Lf), gp,
                                    _i64arr(Lg), _ptr(h), Mv, pp, None, 0, _stream_ptr(stream)))
        return h

    multiconv = hd_multiconv

    def hd_conv_window(self, fs, gs, lo, n, batch=False, M=None, plan=None, h=None, stream=None):
        """Window [lo, lo + n) (per axis) of sum_k fs[k] * gs[k]; fs/gs lists of tensors
        (leading batch axis when batch=True).  See window_for_mode for the paper's modes."""
        N = len(fs)
        nd = self._pairs(fs, gs, batch)
        B = fs[0].shape[0] if batch else 1
        Lf, Lg = list(fs[0].shape[-nd:]), list(gs[0].shape[-nd:])
        h = self._h(h, fs[0], ([B] if batch else []) + [int(v) for v in n])
        fp = (ctypes.c_void_p * N)(*[t.data_ptr() for t in fs])
        gp = (ctypes.c_void_p * N)(*[t.data_ptr() for t in gs])
        Mv = _i64arr(M) if M is not None else None
        pp = ctypes.byref(plan) if plan is not None else None
        self._chk(_lib.hd_conv_window(self.h, _dtype_code(fs[0]), nd, N, B, fp, _i64arr(Lf), gp, _i64arr(Lg),
                                      _ptr(h), Mv, _i64arr(lo), _i64arr(n), pp, None, 0, _stream_ptr(stream)))
        return h

    conv_window = hd_conv_window

    def hd_conv_real(self, f, g, plan=None, h=None, batch=False, stream=None):
        """Full linear convolution of REAL torch tensors (float64 -> complex128
        machinery, float32 -> complex64); leading batch axis when batch=True."""
        import torch
        nd = f.dim() - (1 if batch else 0)
        B = f.shape[0] if batch else 1
        Lf, Lg = list(f.shape[-nd:]), list(g.shape[-nd:])
        if f.dtype == torch.float64:
            dt = HD_C128
        elif f.dtype == torch.float32:
            dt = HD_C64
        else:
            raise TypeError(f"unsupported dtype {f.dtype} (float32 / float64 only)")
        self._arg(f, "f", f.dtype)
        self._arg(g, "g", f.dtype, ([B] if batch else []) + Lg)
        if g.dim() != f.dim():
            raise ValueError("g must have f's number of dims (per-entry g when batch=True)")
        oshape = ([B] if batch else []) + [a + b - 1 for a, b in zip(Lf, Lg)]
        if h is None:
            h = torch.empty(oshape, dtype=f.dtype, device=f.device)
        else:
            self._arg(h, "h", f.dtype, oshape)
        pp = ctypes.byref(plan) if plan is not None else None
        self._chk(_lib.hd_conv_real(self.h, dt, nd, B, _ptr(f), _i64arr(Lf), _ptr(g), _i64arr(Lg), _ptr(h), pp,
                                    _stream_ptr(stream)))
        return h

    conv_real = hd_conv_real

    def hd_conv_explicit(self, fs, gs, plan=None, h=None, stream=None):
        N = len(fs)
        nd = self._pairs(fs, gs)
        Lf, Lg = list(fs[0].shape), list(gs[0].shape)
        h = self._h(h, fs[0], [a + b - 1 for a, b in zip(Lf, Lg)])
        fp = (ctypes.c_void_p * N)(*[t.data_ptr() for t in fs])
        gp = (ctypes.c_void_p * N)(*[t.data_ptr() for t in gs])
        pp = ctypes.byref(plan) if plan is not None else None
        self._chk(_lib.hd_conv_explicit(self.h, _dtype_code(fs[0]), nd, N, fp, _i64arr(Lf), gp,
                                        _i64arr(Lg), _ptr(h), pp, _stream_ptr(stream)))
        return h

    @staticmethod
    def _host_args(fs, gs, h, ndim, batch, plan=None):
        """Validate host operands of hd_conv_host(_async): the library copies exactly
        batch * prod(L) elements of each input and batch * prod(L_out) into h."""
        def info(a, name):
            if isinstance(a, np.ndarray):
                if not a.flags.c_contiguous:
                    raise ValueError(f"{name} must be C-contiguous")
                return str(a.dtype), list(a.shape), a.nbytes, a.ctypes.data
            if not hasattr(a, "data_ptr") or a.device.type != "cpu" or not a.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CPU tensor or numpy array")
            return str(a.dtype).replace("torch.", ""), list(a.shape), a.numel() * a.element_size(), a.data_ptr()
        nd = int(ndim)
        if not 1 <= nd <= 3 or len(fs) != len(gs) or not fs:
            raise ValueError("bad ndim or operand lists")
        dt0, sf, _, _ = info(fs[0], "f[0]")
        if dt0 not in ("complex128", "complex64"):
            raise TypeError(f"unsupported dtype {dt0}")
        esz = 16 if dt0 == "complex128" else 8
        Lf, Lg = sf[-nd:], list(info(gs[0], "g[0]")[1])[-nd:]
        shared = plan is not None and bool(plan.flags & HD_FLAG_SHARED_G)
        nf, ng = int(np.prod(Lf)) * batch, int(np.prod(Lg)) * (1 if shared else batch)
        for k, (f, g) in enumerate(zip(fs, gs)):
            for a, name, n, L in ((f, f"f[{k}]", nf, Lf), (g, f"g[{k}]", ng, Lg)):
                dt, shp, nb, _ = info(a, name)
                if dt != dt0 or shp[-nd:] != L or nb != n * esz:
                    raise ValueError(f"{name}: dtype {dt} shape {shp} does not match f[0] ({dt0}, batch {batch})")
        dth, _, nbh, ptr = info(h, "h")
        nh = batch * int(np.prod([a + b - 1 for a, b in zip(Lf, Lg)]))
        if dth != dt0 or nbh != nh * esz:
            raise ValueError(f"h must hold {nh} {dt0} elements ({nh * esz} bytes), got {dth} with {nbh} bytes")
        return nd, Lf, Lg, (HD_C128 if dt0 == "complex128" else HD_C64), ptr

    def hd_conv_host(self, fs, gs, h, ndim, batch=1, M=None, plan=None, stream=None):
        """End-to-end with HOST buffers: fs, gs lists of (pinned) CPU tensors or numpy
        arrays ([batch] + extents), h a CPU tensor / numpy array receiving the result."""
        N = len(fs)
        def hp(a):
            return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()
        nd, Lf, Lg, dt, _ = self._host_args(fs, gs, h, ndim, batch, plan)
        fp = (ctypes.c_void_p * N)(*[hp(t) for t in fs])
        gp = (ctypes.c_void_p * N)(*[hp(t) for t in gs])
        Mv = _i64arr(M) if M is not None else None
        pp = ctypes.byref(plan) if plan is not None else None
        self._chk(_lib.hd_conv_host(self.h, dt, nd, N, batch, fp, _i64arr(Lf), gp, _i64arr(Lg),
                                    ctypes.c_void_p(hp(h)), Mv, pp, _stream_ptr(stream)))
        return h

    def hd_conv_host_async(self, fs, gs, h, ndim, batch=1, M=None, plan=None):
        """Asynchronous hd_conv_host (triple-buffered context streams): returns after
        enqueueing; the buffers must stay alive and h unread until host_sync()."""
        N = len(fs)
        def hp(a):
            return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()
        nd, Lf, Lg, dt, _ = self._host_args(fs, gs, h, ndim, batch, plan)
        fp = (ctypes.c_void_p * N)(*[hp(t) for t in fs])
        gp = (ctypes.c_void_p * N)(*[hp(t) for t in gs])
        Mv = _i64arr(M) if M is not None else None
        pp = ctypes.byref(plan) if plan is not None else None
        self._chk(_lib.hd_conv_host_async(self.h, dt, nd, N, batch, fp, _i64arr(Lf), gp, _i64arr(Lg),
                                          ctypes.c_void_p(hp(h)), Mv, pp))
        return h

    def host_sync(self):
        self._chk(_lib.hd_host_sync(self.h))

    def hd_forward_residues(self, x, m, q, X=None, stream=None):
        """x: [nlines, L] -> X: [nlines, q*m] (internal residue order)."""
        nl, L = x.shape
        if X is None:
            X = self._out(x, [nl, q * m])
        self._chk(_lib.hd_forward_residues(self.h, _dtype_code(x), nl, _ptr(x), L, m, q, _ptr(X),
                                           _stream_ptr(stream)))
        return X

    def hd_backward_residues(self, X, m, q, Lout, x=None, stream=None):
        nl = X.shape[0]
        if x is None:
            x = self._out(X, [nl, Lout])
        self._chk(_lib.hd_backward_residues(self.h, _dtype_code(X), nl, _ptr(X), m, q, _ptr(x),
                                            Lout, _stream_ptr(stream)))
        return x

    def hd_conv1d_lambda(self, f, g, m, Lambda, M=None, h=None, stream=None):
        """Row f1 (include/hdconv.h): short f [batch, L_f] (* ) long g [batch, L_g] by the
        Lambda > 1 residue matching; returns h [batch, L_f + L_g - 1]."""
        if f.dim() == 1:
            f, g = f.unsqueeze(0), g.unsqueeze(0)
            squeeze = True
        else:
            squeeze = False
        _dtype_code(f)
        if f.dim() != 2 or g.dim() != 2:
            raise ValueError("f, g must be [L] or [batch, L]")
        nb, Lf = f.shape
        Lg = g.shape[1]
        self._arg(f, "f", f.dtype)
        self._arg(g, "g", f.dtype, [nb, Lg])
        h = self._h(h, f, [nb, Lf + Lg - 1])
        self._chk(_lib.hd_conv1d_lambda(self.h, _dtype_code(f), nb, _ptr(f), Lf, _ptr(g), Lg, _ptr(h),
                                        0 if M is None else int(M), int(m), int(Lambda), _stream_ptr(stream)))
        return h[0] if squeeze else h

    conv1d_lambda = hd_conv1d_lambda

    def default_plan(self, dtype, Lf, Lg, M=None, npairs=1):
        return hd_plan_default(dtype, Lf, Lg, M, npairs)

    def hd_tune(self, dtype, Lf, Lg, M=None, N=1, batch=1, exhaustive=False, reps=5, stream=None):
        p = Plan()
        Mv = _i64arr(M) if M is not None else None
        self._chk(_lib.hd_tune(self.h, dtype, len(Lf), N, batch, _i64arr(Lf), _i64arr(Lg), Mv,
                               HD_TUNE_EXHAUSTIVE if exhaustive else HD_TUNE_PER_AXIS, reps,
                               _stream_ptr(stream), ctypes.byref(p)))
        return p

    tune = hd_tune

    def tune_explicit(self, dtype, Lf, Lg, N=1, reps=3, stream=None):
        """hd_tune_explicit: the explicit-padding baseline's own tuned plan (cached for
        hd_conv_explicit(plan=None))."""
        p = Plan()
        self._chk(_lib.hd_tune_explicit(self.h, dtype, len(Lf), N, _i64arr(Lf), _i64arr(Lg), reps,
                                        _stream_ptr(stream), ctypes.byref(p)))
        return p

    def hd_tune_ex(self, dtype, Lf, Lg, M=None, N=1, batch=1, mode="per_axis", n1=16, seed=0,
                   proxy_rows=0, reps=5, fake_cost=0, stream=None):
        """Extended tuner: mode per_axis | exhaustive | random (A1, n1 samples, seed);
        proxy_rows > 0 tunes the axes other than 0 on the skinny proxy problem."""
        flags = {"per_axis": HD_TUNE_PER_AXIS, "exhaustive": HD_TUNE_EXHAUSTIVE, "random": HD_TUNE_RANDOM}[mode]
        o = TuneOpts(flags=flags, reps=reps, n1=n1, fake_cost=fake_cost, seed=seed, proxy_rows=proxy_rows)
        p = Plan()
        Mv = _i64arr(M) if M is not None else None
        self._chk(_lib.hd_tune_ex(self.h, dtype, len(Lf), N, batch, _i64arr(Lf), _i64arr(Lg), Mv,
                                  ctypes.byref(o), _stream_ptr(stream), ctypes.byref(p)))
        return p

    def hd_tune_log(self):
        n = _lib.hd_tune_log(self.h, 0, None, None)
        plans = (Plan * max(n, 1))()
        secs = np.zeros(max(n, 1), dtype=np.float64)
        _lib.hd_tune_log(self.h, n, plans, secs.ctypes.data_as(ctypes.c_void_p))
        return [(plans[i], float(secs[i])) for i in range(n)]

    def hd_workspace_bytes(self, dtype, Lf, Lg, M=None, npairs=1, batch=1, plan=None):
        Mv = _i64arr(M) if M is not None else None
        pp = ctypes.byref(plan) if plan is not None else None
        return _lib.hd_workspace_bytes(self.h, dtype, len(Lf), npairs, batch, _i64arr(Lf),
                                       _i64arr(Lg), Mv, pp)

    def profile_enable(self, on=True):
        self._chk(_lib.hd_profile_enable(self.h, 1 if on else 0))

    def profile_reset(self):
        self._chk(_lib.hd_profile_reset(self.h))

    def profile_read(self):
        n = _lib.hd_profile_read(self.h, 0, None, None, None)
        ms = np.zeros(max(n, 1))
        la = np.zeros(max(n, 1), dtype=np.int64)
        names = ctypes.create_string_buffer(32 * max(n, 1))
        _lib.hd_profile_read(self.h, n, ms.ctypes.data_as(ctypes.c_void_p),
                             la.ctypes.data_as(ctypes.c_void_p), names)
        out = {}
        for i in range(n):
            nm = names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(la[i]))
        return out

    def launch_count(self):
        return int(_lib.hd_launch_count(self.h))

    def graph_replays(self):
        """Calls served by a captured CUDA graph (HD_FLAG_GRAPH)."""
        return int(_lib.hd_graph_replays(self.h))

    def engine_launches(self, engine):
        """Pass launches on one engine (HD_ENGINE_*) since the context was created."""
        return int(_lib.hd_engine_launches(self.h, engine))

    # ---- multi-GPU (include/hdconv.h "multi-GPU"): NCCL inside libhdconv ---------
    def dist_init(self, group=None):
        """Create this context's NCCL communicator over the torch.distributed group: rank
        0 draws the unique id (hd_dist_unique_id) and the group broadcasts it (the only
        Python-side step); a group of one needs no NCCL."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if world > 1:
            if rank == 0:
                _check_dist(_lib.hd_dist_unique_id(uid))
            obj = [bytes(uid.raw)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        _check_dist(_lib.hd_dist_init(self.h, uid, world, rank))
        self.world, self.rank = world, rank
        return world, rank

    def conv1d_dist(self, f, g, batch, shard=HD_SHARD_BATCH, plan=None, h=None, stream=None):
        """1-D batch of pairs over the ranks (hd_conv1d_dist): HD_SHARD_BATCH with f, g this
        rank's slice; HD_SHARD_RESIDUE with f, g the whole batch.  Returns this rank's rows."""
        Lf, Lg = f.shape[-1], g.shape[-1]
        lo, hi = dist_partition(batch, self.world, self.rank)
        nb = hi - lo if shard == HD_SHARD_BATCH else batch
        self._arg(f, "f", f.dtype, [nb, Lf])
        self._arg(g, "g", f.dtype, [nb, Lg])
        h = self._h(h, f, [hi - lo, Lf + Lg - 1])
        pp = ctypes.byref(plan) if plan is not None else None
        _check_dist(_lib.hd_conv1d_dist(self.h, _dtype_code(f), int(batch), _ptr(f), Lf, _ptr(g), Lg, _ptr(h), pp,
                                        int(shard), _stream_ptr(stream)), self.h)
        return h

    def slab(self, dtype, Lf, Lg, nchunks=0, plan=None):
        return slab_plan(dtype, Lf, Lg, self.world, self.rank, nchunks, plan)

    def conv2d_dist(self, f_rows, g, Lf, plan=None, nchunks=0, h=None, stream=None):
        """This rank's output rows of f * g with f row-slab decomposed (hd_conv2d_dist);
        f_rows = rows [in_lo, in_hi) of f (Lf: global extents), g replicated."""
        dt = _dtype_code(g)
        Lg = list(g.shape)
        sp = self.slab(dt, Lf, Lg, nchunks, plan)
        self._arg(f_rows, "f_rows", g.dtype, [sp.in_hi - sp.in_lo, Lf[1]])
        self._arg(g, "g", g.dtype)
        h = self._h(h, g, [sp.out_hi - sp.out_lo, Lf[1] + Lg[1] - 1])
        pp = ctypes.byref(plan) if plan is not None else None
        _check_dist(_lib.hd_conv2d_dist(self.h, dt, _ptr(f_rows), _i64arr(Lf), _ptr(g), _i64arr(Lg), _ptr(h), pp,
                                        int(nchunks), _stream_ptr(stream)), self.h)
        return h

    def conv3d_dist(self, f_planes, g, Lf, plan=None, h=None, stream=None):
        """This rank's output planes of f * g with f z-slab decomposed (hd_conv3d_dist)."""
        dt = _dtype_code(g)
        Lg = list(g.shape)
        sp = self.slab(dt, Lf, Lg, 1, plan)
        self._arg(f_planes, "f_planes", g.dtype, [sp.in_hi - sp.in_lo, Lf[1], Lf[2]])
        self._arg(g, "g", g.dtype)
        h = self._h(h, g, [sp.out_hi - sp.out_lo] + [a + b - 1 for a, b in zip(Lf[1:], Lg[1:])])
        pp = ctypes.byref(plan) if plan is not None else None
        _check_dist(_lib.hd_conv3d_dist(self.h, dt, _ptr(f_planes), _i64arr(Lf), _ptr(g), _i64arr(Lg), _ptr(h), pp,
                                        _stream_ptr(stream)), self.h)
        return h

    def filter_image(self, img, kernel, window=None, channel_last=True, out=None, stream=None):
        """The paper's image filter (hd_filter_image): every channel of the real image
        `img` ([H][W][C] or [C][H][W]) convolved with dictionary kernel `kernel` (id or
        name), real part, window (lo, n) of the full result (None: all)."""
        import torch
        kid = FILTER_NAMES.index(kernel) if isinstance(kernel, str) else int(kernel)
        if img.dtype == torch.float64:
            dt = HD_C128
        elif img.dtype == torch.float32:
            dt = HD_C64
        else:
            raise TypeError("img must be float64 or float32")
        if img.dim() != 3:
            raise ValueError("img must be [H][W][C] or [C][H][W]")
        H, W, C = (img.shape[0], img.shape[1], img.shape[2]) if channel_last else (img.shape[1], img.shape[2],
                                                                                   img.shape[0])
        self._arg(img, "img", img.dtype)
        n = filter_kernel(kid)[1].shape[0]
        lo, nn = (window if window is not None else ([0, 0], [H + n - 1, W + n - 1]))
        shape = [nn[0], nn[1], C] if channel_last else [C, nn[0], nn[1]]
        out = self._h(out, img, shape)
        st = _lib.hd_filter_image(self.h, dt, _ptr(img), H, W, C, 1 if channel_last else 0, kid, _i64arr(lo),
                                  _i64arr(nn), _ptr(out), _stream_ptr(stream))
        if st != HD_OK:
            raise HDError(st, (_lib.hd_filter_last_error() or b"").decode())
        return out

    def slab_stage(self, dtype, sp, Lf, Lg, stage, inp, out, gt=None, scratch=None, stream=None):
        """One compute stage of a slab decomposition (hd_slab_stage), no exchange."""
        p = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _check_dist(_lib.hd_slab_stage(self.h, dtype, ctypes.byref(sp), _i64arr(Lf), _i64arr(Lg), int(stage),
                                       p(inp), p(gt), p(out), p(scratch), _stream_ptr(stream)), self.h)
        return out

    def hd_pass(self, dtype, desc, stream=None):
        """One pass with explicit layouts (include/hdconv.h hd_pass)."""
        self._chk(_lib.hd_pass(self.h, dtype, ctypes.byref(desc), _stream_ptr(stream)))
