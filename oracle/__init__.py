"""CPU oracle for hybrid-dealiased convolution (arXiv 2306.10016).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
path (paper_2306_10016_b200/, libhdconv.so) never imports it, and the two
share no code (see oracle/oracle.c header).

Every function is the plain definition the method reaches (PAPER.md:537-541
Eq. 4 linear convolution; Eq. 1 DFT) and cites its passage.
Floating point is complex double; complex64 inputs are upcast exactly.

Parity pins: tests/test_oracle.py checks every function here against values
and identities that do not come from this module (numpy.fft circular
convolution, numpy/scipy integer convolution, golden worked examples with
citations, delta/shift/commutativity/separability identities, the generating
polynomial identity).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc + OpenMP (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            lib.oracle_multiconv.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P, P]
            lib.oracle_multiconv_sampled.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P,
                                                     I64, P, P]
            lib.oracle_dft.argtypes = [I64, I64, P, ctypes.c_int, P]
            lib.oracle_poly_eval.argtypes = [ctypes.c_int, P, P, I64, P, P]
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_poly_eps.restype = ctypes.c_double
            _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex128)


def _i64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def multiconv(fs, gs) -> np.ndarray:
    """h = sum_k f_k * g_k (Eq. 4 per axis; multi-convolution
    reading R9).  All f_k share one shape, all g_k another; ndim in {1,2,3}.
    Output extent Lf_i + Lg_i - 1 per axis (reading R3)."""
    fs = [_c128(f) for f in fs]
    gs = [_c128(g) for g in gs]
    n = len(fs)
    assert n == len(gs) and n >= 1
    ndim = fs[0].ndim
    assert 1 <= ndim <= 3 and all(f.shape == fs[0].shape for f in fs)
    assert all(g.shape == gs[0].shape and g.ndim == ndim for g in gs)
    Lf, Lg = _i64(fs[0].shape), _i64(gs[0].shape)
    out = np.zeros(tuple(int(a + b - 1) for a, b in zip(Lf, Lg)), dtype=np.complex128)
    fp = (ctypes.c_void_p * n)(*[f.ctypes.data for f in fs])
    gp = (ctypes.c_void_p * n)(*[g.ctypes.data for g in gs])
    rc = _load().oracle_multiconv(ndim, n, _ptr(Lf), fp, _ptr(Lg), gp, _ptr(out))
    if rc != 0:
        raise ValueError("oracle_multiconv rejected its arguments")
    return out


def conv(f, g) -> np.ndarray:
    """Full linear convolution f * g (Eq. 4), 1-3 dims."""
    return multiconv([f], [g])


def conv_batch(f, g) -> np.ndarray:
    """Independent pairs along axis 0 (config 2 reading R19)."""
    return np.stack([conv(f[b], g[b]) for b in range(f.shape[0])])


def multiconv_sampled(fs, gs, idx) -> np.ndarray:
    """sum_k (f_k * g_k)[o] at the output indices idx[s, :] (same formula)."""
    fs = [_c128(f) for f in fs]
    gs = [_c128(g) for g in gs]
    n = len(fs)
    ndim = fs[0].ndim
    idx = _i64(idx).reshape(-1, ndim)
    out = np.zeros(idx.shape[0], dtype=np.complex128)
    Lf, Lg = _i64(fs[0].shape), _i64(gs[0].shape)
    fp = (ctypes.c_void_p * n)(*[f.ctypes.data for f in fs])
    gp = (ctypes.c_void_p * n)(*[g.ctypes.data for g in gs])
    rc = _load().oracle_multiconv_sampled(ndim, n, _ptr(Lf), fp, _ptr(Lg), gp,
                                          idx.shape[0], _ptr(idx), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_multiconv_sampled rejected its arguments")
    return out


def conv_sampled(f, g, idx) -> np.ndarray:
    return multiconv_sampled([f], [g], idx)


def dft(x, M: int, sign: int = +1) -> np.ndarray:
    """Naive DFT of x zero-padded to M, X_k = sum_j zeta_M^{sign k j} x_j,
    zeta_M = exp(2 pi i/M) (Eq. 1, positive exponent forward,
    unnormalised; reading R1/R2)."""
    x = _c128(x).ravel()
    out = np.zeros(M, dtype=np.complex128)
    rc = _load().oracle_dft(int(M), x.size, _ptr(x), int(sign), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_dft rejected its arguments")
    return out


def residue_block(x, m: int, q: int, r: int) -> np.ndarray:
    """Residue r of the implicitly padded transform: F_{q l + r}, l < m, of x
    zero-padded to M1 = q m (k = q l + r, Forward Eq.)."""
    return dft(x, q * m, +1)[r::q]


def lambda_conv(f, g, m: int, Lam: int, M: int | None = None) -> np.ndarray:
    """Linear convolution of a short f and a long g by the Lambda > 1 residue
    matching of PAPER.md:680-702 (Final Algorithm For One Dimension), written out
    step by step in the paper's notation with naive DFTs (slow; small sizes only):

      p_f = ceil(L_f / m), p_g = ceil(L_g / (Lam m)), q_g = ceil(M / (Lam m)),
      q_f = Lam q_g; M1 = q_g Lam m = q_f m;
      F_{r_f}[l_f] = F_{q_f l_f + r_f} (size-m residues of f),
      G_{r_g}[l_g] = G_{q_g l_g + r_g} (size-Lam m residues of g);
      for l_g < Lam m: l_f = floor(l_g / Lam), lambda = l_g mod Lam,
      r_f = q_g lambda + r_g, so q_g l_g + r_g = q_f l_f + r_f;
      H_{r_g}[l_g] = F_{r_f}[l_f] G_{r_g}[l_g] (the product of matching
      residues), h_k = (1/M1) sum_{r_g, l_g} zeta_{M1}^{-k (q_g l_g + r_g)} H_{r_g}[l_g]
      (Backward Eq. PAPER.md:531 with q_g, Lam m), k < L_f + L_g - 1.

    Requires L_f <= L_g (the larger array is called g)."""
    f = _c128(f).ravel()
    g = _c128(g).ravel()
    Lf, Lg = f.size, g.size
    if Lf > Lg:
        raise ValueError("lambda_conv needs L_f <= L_g (PAPER.md:682)")
    Lout = Lf + Lg - 1
    M = Lout if M is None else int(M)
    qg = -(-M // (Lam * m))
    qf = Lam * qg
    M1 = qg * Lam * m
    if -(-Lf // m) > qf or -(-Lg // (Lam * m)) > qg:
        raise ValueError("inputs longer than M1")
    F = [residue_block(f, m, qf, rf) for rf in range(qf)]          # F_{r_f}[l_f]
    G = [residue_block(g, Lam * m, qg, rg) for rg in range(qg)]    # G_{r_g}[l_g]
    S = np.zeros(M1, dtype=np.complex128)                          # spectrum at q_g l_g + r_g
    for rg in range(qg):
        for lg in range(Lam * m):
            lf, lam = lg // Lam, lg % Lam
            rf = qg * lam + rg
            S[qg * lg + rg] = F[rf][lf] * G[rg][lg]
    h = dft(S, M1, -1) / M1
    return h[:Lout]


def poly_eps() -> float:
    """Unit roundoff of poly_eval's accumulation (long double in oracle.c)."""
    return float(_load().oracle_poly_eps())


def poly_eval(a, z) -> np.ndarray:
    """P_a(z) = sum_o a[o] prod_i z_i^{o_i} at points z[p, :] (nested Horner,
    accumulated in long double, rounded to double once)."""
    a = _c128(a)
    ndim = a.ndim
    z = _c128(z).reshape(-1, ndim)
    out = np.zeros(z.shape[0], dtype=np.complex128)
    L = _i64(a.shape)
    rc = _load().oracle_poly_eval(ndim, _ptr(L), _ptr(a), z.shape[0], _ptr(z), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_poly_eval rejected its arguments")
    return out


def alias_fold(h_full: np.ndarray, M1) -> np.ndarray:
    """Output of an undersized transform (M1 < L_out on an axis): the M1-periodic
    fold sum_s (f*g)_{k + s M1} (the s != 0 alias terms;
    SPEC.md:154 worked example).  Plain definition on top of conv()."""
    h = np.asarray(h_full)
    M1 = [int(v) for v in np.atleast_1d(M1)]
    for ax, M in enumerate(M1):
        n = h.shape[ax]
        if M >= n:
            continue
        nb = -(-n // M)
        pad = [(0, 0)] * h.ndim
        pad[ax] = (0, nb * M - n)
        hp = np.pad(h, pad)
        shp = list(h.shape)
        shp[ax:ax + 1] = [nb, M]
        h = hp.reshape(shp).sum(axis=ax)
    return h


def rel_l2(a, b) -> float:
    """||a - b||_2 / ||b||_2 (parity metric)."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    nb = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0))
