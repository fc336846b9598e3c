"""Pins for the CPU oracle (oracle/).  CPU only (-m "not gpu").

Every check compares the oracle with something other than itself:
golden worked examples (tests/golden/*.json, each with its citation),
numpy.fft circular convolution with M >= L_out (the convolution theorem,
PAPER.md:545-549), exact integer convolution from numpy/scipy, and identities
(delta, shift, commutativity, separability, generating polynomial).
"""
import numpy as np
import pytest
import scipy.signal

import oracle
import synth


def _np_circular_conv(f, g, M):
    """Convolution theorem with explicit padding to M, numpy FFT."""
    axes = tuple(range(f.ndim))
    F = np.fft.fftn(f, s=M, axes=axes)
    G = np.fft.fftn(g, s=M, axes=axes)
    return np.fft.ifftn(F * G, axes=axes)


def _int_conv(a, b):
    """Exact complex integer convolution from integer library convolutions."""
    ar, ai = np.real(a).astype(np.int64), np.imag(a).astype(np.int64)
    br, bi = np.real(b).astype(np.int64), np.imag(b).astype(np.int64)
    cv = lambda x, y: scipy.signal.convolve(x, y, mode="full", method="direct")
    return cv(ar, br) - cv(ai, bi), cv(ar, bi) + cv(ai, br)


def test_splitmix64_reference_sequence():
    # splitmix64 with state 0: the published first outputs of the generator
    s = synth.Stream(0)
    i = np.arange(1, 4, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = synth._mix64(np.uint64(0) + i * synth.GOLDEN)
    assert int(x[0]) == 0xE220A8397B1DCDAF
    assert int(x[1]) == 0x6E789E6AA1B965F4
    assert int(x[2]) == 0x06C45D188009454F
    u = s.uniform(3)
    assert np.all((u >= 0) & (u < 1))
    assert u[0] == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53


def test_worked_example_1d(golden):
    d = golden("worked_example_1d.json")
    h = oracle.conv(np.array(d["f"], complex), np.array(d["g"], complex))
    assert np.array_equal(h, np.array(d["h"], complex))


def test_worked_example_2d_ones(golden):
    d = golden("conv2d_ones.json")
    h = oracle.conv(np.array(d["f"], complex), np.array(d["g"], complex))
    assert np.array_equal(h, np.array(d["h"], complex))


def test_alias_fold_golden(golden):
    d = golden("alias_fold_1d.json")
    h = oracle.conv(np.array(d["f"], complex), np.array(d["g"], complex))
    a = oracle.alias_fold(h, d["M"])
    assert np.array_equal(a, np.array(d["h"], complex))
    # and it is the undersized explicit transform (numpy FFT of size M)
    ref = _np_circular_conv(np.array(d["f"], complex), np.array(d["g"], complex), (d["M"],))
    assert np.allclose(a, ref, atol=1e-12)


def test_residue_forward_golden(golden):
    d = golden("residue_forward.json")
    x = np.array(d["x"], complex)
    for r in (0, 1):
        want = np.array([complex(a, b) for a, b in d[f"r{r}"]])
        got = oracle.residue_block(x, d["m"], d["q"], r)
        assert np.allclose(got, want, atol=1e-13)


@pytest.mark.parametrize("M", [1, 2, 3, 5, 8, 12, 31, 64])
def test_dft_orthogonality(M):
    # sum_j zeta_M^{l j} = M if l = 0 mod M else 0
    X = oracle.dft(np.ones(M), M, +1)
    want = np.zeros(M, complex)
    want[0] = M
    assert np.allclose(X, want, atol=1e-12 * M)
    Xm = oracle.dft(np.ones(M), M, -1)
    assert np.allclose(Xm, want, atol=1e-12 * M)


@pytest.mark.parametrize("M,L", [(1, 1), (4, 3), (7, 7), (16, 9), (45, 20), (128, 100)])
def test_dft_matches_numpy(M, L):
    x, _ = synth.random_pair(M * 31 + L, (L,), (1,))
    xp = np.zeros(M, complex)
    xp[:L] = x
    # paper forward (positive exponent, unnormalised) == M * numpy ifft
    assert np.allclose(oracle.dft(x, M, +1), M * np.fft.ifft(xp), atol=1e-12 * M)
    assert np.allclose(oracle.dft(x, M, -1), np.fft.fft(xp), atol=1e-12 * M)


def test_residue_blocks_cover_the_spectrum():
    # k = q l + r is a bijection of [0, qm)
    x, _ = synth.random_pair(5, (13,), (1,))
    m, q = 4, 5
    full = M_x = np.fft.ifft(np.concatenate([x, np.zeros(q * m - 13)])) * (q * m)
    re = np.zeros(q * m, complex)
    for r in range(q):
        re[r::q] = oracle.residue_block(x, m, q, r)
    assert np.allclose(re, full, atol=1e-12)
    del M_x


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_brute_force_fft_convolution(ndim):
    # O1: oracle == numpy FFT convolution padded to M >= L_out, many tiny shapes
    rng_seed = 100 * ndim
    cases = 12 if ndim < 3 else 6
    for c in range(cases):
        s = synth.Stream(rng_seed + c)
        lim = {1: 24, 2: 10, 3: 6}[ndim]
        Lf = tuple(1 + int(v * lim) for v in s.uniform(ndim))
        Lg = tuple(1 + int(v * lim) for v in s.uniform(ndim))
        f, g = synth.random_pair(rng_seed + 1000 + c, Lf, Lg)
        Lout = tuple(a + b - 1 for a, b in zip(Lf, Lg))
        M = tuple(o + int(v * 5) for o, v in zip(Lout, s.uniform(ndim)))
        ref = _np_circular_conv(f, g, M)[tuple(slice(0, o) for o in Lout)]
        h = oracle.conv(f, g)
        assert h.shape == Lout
        assert oracle.rel_l2(h, ref) < 1e-13
        # zero tail of the padded explicit result (padding monotonicity)
        full = _np_circular_conv(f, g, M)
        tail = full.copy()
        tail[tuple(slice(0, o) for o in Lout)] = 0
        assert np.max(np.abs(tail)) < 1e-12


def test_delta_identity_and_shift():
    # O3: delta_0 * g = g, delta_k shifts by k
    _, g = synth.random_pair(7, (1,), (9,))
    assert np.array_equal(oracle.conv(np.array([1 + 0j]), g), g)
    d = np.zeros(4, complex)
    d[3] = 1
    h = oracle.conv(d, g)
    assert np.array_equal(h[3:], g) and np.all(h[:3] == 0)
    _, g2 = synth.random_pair(8, (1, 1), (5, 6))
    d2 = np.zeros((2, 3), complex)
    d2[1, 2] = 1
    h2 = oracle.conv(d2, g2)
    assert np.array_equal(h2[1:, 2:], g2)
    assert np.all(h2[0, :] == 0) and np.all(h2[:, :2] == 0)
    _, g3 = synth.random_pair(9, (1,), (3, 4, 5))
    d3 = np.zeros((1, 1, 1), complex)
    d3[0, 0, 0] = 1
    assert np.array_equal(oracle.conv(d3, g3), g3)


def test_commutativity():
    # O4: f * g = g * f
    for ndim, (sf, sg) in {1: ((17,), (5,)), 2: ((6, 9), (4, 3)), 3: ((3, 4, 5), (2, 5, 3))}.items():
        f, g = synth.random_pair(11 + ndim, sf, sg)
        assert oracle.rel_l2(oracle.conv(f, g), oracle.conv(g, f)) < 1e-15


def test_separability():
    # O5: rank-1 inputs give the outer product of 1D convolutions (numpy.convolve)
    s = synth.Stream(21)
    a, b, c = (s.complex_uniform((n,)) for n in (7, 5, 4))
    d, e, w = (s.complex_uniform((n,)) for n in (3, 6, 2))
    f2 = np.outer(a, b)
    g2 = np.outer(d, e)
    h2 = oracle.conv(f2, g2)
    assert oracle.rel_l2(h2, np.outer(np.convolve(a, d), np.convolve(b, e))) < 1e-14
    f3 = np.einsum("i,j,k->ijk", a, b, c)
    g3 = np.einsum("i,j,k->ijk", d, e, w)
    want = np.einsum("i,j,k->ijk", np.convolve(a, d), np.convolve(b, e), np.convolve(c, w))
    assert oracle.rel_l2(oracle.conv(f3, g3), want) < 1e-14


@pytest.mark.parametrize("sf,sg", [((40,), (33,)), ((9, 12), (7, 5)), ((5, 6, 4), (3, 4, 5))])
def test_integer_exactness(sf, sg):
    # O6: integer inputs in [-8, 8] give exactly the integer convolution
    f, g = synth.integer_pair(31, sf, sg)
    re, im = _int_conv(f, g)
    h = oracle.conv(f, g)
    assert np.array_equal(h.real, re.astype(float))
    assert np.array_equal(h.imag, im.astype(float))


def test_sum_and_polynomial_identity():
    # O7: sum h = sum f * sum g; P_h(z) = P_f(z) P_g(z) on the unit torus
    f, g = synth.random_pair(41, (6, 7), (5, 3))
    h = oracle.conv(f, g)
    assert abs(h.sum() - f.sum() * g.sum()) < 1e-12 * np.abs(h).sum()
    z = synth.unit_torus_points(8, 2)
    Ph = oracle.poly_eval(h, z)
    Pf = np.array([np.polynomial.polynomial.polyval2d(p[0], p[1], f) for p in z])
    Pg = np.array([np.polynomial.polynomial.polyval2d(p[0], p[1], g) for p in z])
    assert np.allclose(Ph, Pf * Pg, atol=1e-12 * np.linalg.norm(h))
    # poly_eval itself agrees with numpy polyval (1D and 3D)
    f1, _ = synth.random_pair(42, (11,), (1,))
    z1 = synth.unit_torus_points(5, 1)
    assert np.allclose(oracle.poly_eval(f1, z1),
                       np.polynomial.polynomial.polyval(z1[:, 0], f1), atol=1e-13)
    f3, _ = synth.random_pair(43, (3, 2, 4), (1,))
    z3 = synth.unit_torus_points(4, 3)
    want = [np.polynomial.polynomial.polyval3d(p[0], p[1], p[2], f3) for p in z3]
    assert np.allclose(oracle.poly_eval(f3, z3), want, atol=1e-13)


def test_multiconv_is_sum_of_pairs():
    s = synth.Stream(51)
    fs = [s.complex_uniform((5, 8)) for _ in range(3)]
    gs = [s.complex_uniform((4, 3)) for _ in range(3)]
    h = oracle.multiconv(fs, gs)
    ref = sum(_np_circular_conv(f, g, (8, 10)) for f, g in zip(fs, gs))[:8, :10]
    assert oracle.rel_l2(h, ref) < 1e-13


def test_sampled_matches_full():
    f, g = synth.random_pair(61, (9, 13), (6, 4))
    h = oracle.conv(f, g)
    idx = synth.sample_indices(h.shape, n_random=50)
    v = oracle.conv_sampled(f, g, idx)
    assert np.array_equal(v, h[idx[:, 0], idx[:, 1]])
    f3, g3 = synth.random_pair(62, (4, 5, 3), (3, 2, 6))
    h3 = oracle.conv(f3, g3)
    idx3 = synth.sample_indices(h3.shape, n_random=30)
    assert np.array_equal(oracle.conv_sampled(f3, g3, idx3), h3[tuple(idx3.T)])


def test_rejects_bad_arguments():
    with pytest.raises(ValueError):
        oracle.conv_sampled(np.ones(3, complex), np.ones(2, complex), np.array([[4]]))
    with pytest.raises(ValueError):
        oracle.dft(np.ones(5), 3)


def test_config_inputs_recipe():
    d = synth.config_inputs(1)
    f, g = d["f"][0], d["g"][0]
    assert f.shape == (64,) and g.shape == (40,)
    assert np.all(np.abs(f.real) <= 1) and np.all(np.abs(g.imag) <= 1)
    # f then g from one stream: g continues f's counter
    s = synth.Stream(0)
    s.uniform(128)
    u = s.uniform(2)
    assert g[0] == complex(-1 + 2 * u[0], -1 + 2 * u[1])
    d3 = synth.config_inputs(3, scale=16)
    assert np.all(d3["f"][0].imag == 0)


@pytest.mark.parametrize("Lf,Lg,m,Lam,M", [(7, 30, 4, 2, None), (13, 50, 4, 4, None), (5, 21, 2, 8, 40),
                                           (16, 16, 4, 2, None), (1, 9, 2, 2, None), (30, 100, 8, 2, 160)])
def test_lambda_conv_matches_numpy(Lf, Lg, m, Lam, M):
    # f1: the Lambda > 1 residue matching reaches the linear
    # convolution: compare with numpy's direct convolution (not the oracle's C code)
    f, g = synth.random_pair(60 + Lf, (Lf,), (Lg,))
    h = oracle.lambda_conv(f, g, m, Lam, M)
    assert oracle.rel_l2(h, np.convolve(f, g)) < 1e-12


def test_lambda_index_map_is_a_bijection():
    # q_g l_g + r_g = q_f l_f + r_f with l_f = floor(l_g / Lam),
    # lambda = l_g mod Lam, r_f = q_g lambda + r_g covers every frequency of M1 once
    for qg, Lam, m in [(3, 2, 4), (5, 4, 8), (1, 8, 2), (9, 2, 16)]:
        qf = Lam * qg
        seen = set()
        for rg in range(qg):
            for lg in range(Lam * m):
                lf, lam = lg // Lam, lg % Lam
                rf = qg * lam + rg
                assert 0 <= rf < qf and 0 <= lf < m
                assert qg * lg + rg == qf * lf + rf
                seen.add(qf * lf + rf)
        assert seen == set(range(qg * Lam * m))


def test_lambda_conv_integer_exact_and_rejects_swapped():
    f, g = synth.integer_pair(62, (9,), (40,))
    re, im = _int_conv(f, g)
    h = oracle.lambda_conv(f, g, 4, 2)
    assert np.abs(h.real - re).max() < 1e-9 and np.abs(h.imag - im).max() < 1e-9
    with pytest.raises(ValueError):
        oracle.lambda_conv(g, f, 4, 2)
