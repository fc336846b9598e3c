"""Tuner heuristics.

CPU: the record-analysis helpers against the worked values of SPEC.md:364-409.
GPU: hd_tune_ex's search logic with the cost-injection hook (deterministic costs,
no timing noise): random search with n1 >= |space| equals the grid search, a fixed
seed is repeatable, ties break lexicographically, and the skinny proxy returns an
admissible plan that convolves correctly."""
import pytest

import oracle
import synth


@pytest.fixture(scope="module")
def H():
    from paper_2306_10016_b200 import hdconv
    return hdconv


def test_sort_lists_topk(H):
    assert H.sort_lists_topk([8, 16, 32], [3.0, 1.0, 2.0], 1) == ([16], [1.0], [1])
    a, b, i = H.sort_lists_topk([8, 16, 32], [3.0, 1.0, 2.0], 3)
    assert a == [16, 32, 8] and b == [1.0, 2.0, 3.0] and i == [1, 2, 0]
    assert H.sort_lists_topk([8, 16], [1.0, 2.0], 0) == ([], [], [])
    with pytest.raises(ValueError):
        H.sort_lists_topk([1], [1.0, 2.0], 1)


def test_sort_lists_eps(H):
    # T = 1 + 0.5 * (3 - 1) = 2 -> {16: 0, 32: 0.5}
    assert H.sort_lists_eps([8, 16, 32], [3.0, 1.0, 2.0], 0.5) == ([16, 32], [0.0, 0.5])
    a, b = H.sort_lists_eps([8, 16, 32], [3.0, 1.0, 2.0], 1.0)
    assert a == [16, 32, 8] and b == [0.0, 0.5, 1.0]
    assert H.sort_lists_eps([8, 16, 32], [3.0, 1.0, 2.0], 0.0) == ([16], [0.0])
    assert H.sort_lists_eps([4, 5], [2.0, 2.0], 0.3) == ([4, 5], [0.0, 0.0])
    with pytest.raises(ValueError):
        H.sort_lists_eps([], [], 0.5)


def test_epsilon_smallest_rectangle(H):
    square = ([16, 32, 64], [5.0, 4.0, 6.0])  # m* = 32
    rects = {8: ([16, 64], [1.0, 2.0]), 32: ([32, 64], [1.0, 2.0])}
    assert H.epsilon_smallest_rectangle(square, rects, 1.0) == 32
    same = {4: ([32, 8], [1.0, 3.0]), 16: ([32], [1.0])}
    assert H.epsilon_smallest_rectangle(square, same, 0.0) == 4
    assert H.epsilon_smallest_rectangle(square, {8: ([16, 32], [1.0, 2.0])}, 0.0) is None


def test_skinny_estimate(H):
    assert H.skinny_estimate(([16, 32], [5.0, 4.0]), ([16, 8], [1.0, 2.0])) == (16, 5.0, 32, 4.0)
    assert H.skinny_estimate(([16, 32], [5.0, 4.0]), ([32], [1.0])) == (32, 4.0, 32, 4.0)
    assert H.skinny_estimate(([16, 32], [5.0, 4.0]), ([128], [1.0]))[0] == "miss"


# ---------------------------------------------------------------- device-side search
def _key(p, nd):
    return tuple((p.axis[i].m, p.axis[i].C, p.axis[i].S, p.axis[i].D, p.axis[i].threads) for i in range(nd))


@pytest.fixture(scope="module")
def ctx(H):
    pytest.importorskip("torch")
    c = H.Context(0)
    yield c
    c.close()


@pytest.mark.gpu
def test_random_search_covers_grid_search(ctx, H):
    Lf, Lg = [40, 30], [5, 6]
    ex = ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="exhaustive", fake_cost=1, seed=5)
    n_space = len(ctx.hd_tune_log())
    rnd = ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="random", n1=n_space + 10, fake_cost=1, seed=5)
    assert _key(rnd, 2) == _key(ex, 2)
    assert len(ctx.hd_tune_log()) == n_space


@pytest.mark.gpu
def test_random_search_is_seeded(ctx, H):
    Lf, Lg = [40, 30], [5, 6]
    a = ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="random", n1=7, fake_cost=1, seed=11)
    la = [_key(p, 2) for p, _ in ctx.hd_tune_log()]
    b = ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="random", n1=7, fake_cost=1, seed=11)
    lb = [_key(p, 2) for p, _ in ctx.hd_tune_log()]
    assert la == lb and len(la) == 7 and _key(a, 2) == _key(b, 2)
    # the winner is the argmin of the sampled costs
    log = ctx.hd_tune_log()
    assert abs(min(t for _, t in log) - b.tuned_seconds) < 1e-15


@pytest.mark.gpu
def test_ties_break_lexicographically(ctx, H):
    Lf, Lg = [40, 30], [5, 6]
    p = ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="exhaustive", fake_cost=2)
    keys = [_key(q, 2) for q, _ in ctx.hd_tune_log()]
    assert _key(p, 2) == min(keys)


@pytest.mark.gpu
def test_skinny_proxy_tuning(ctx, H):
    import torch
    Lf, Lg = [300, 260], [31, 17]
    p = ctx.hd_tune_ex(H.HD_C128, Lf, Lg, proxy_rows=32, reps=2)
    assert p.tuned_seconds > 0
    f, g = synth.random_pair(790, tuple(Lf), tuple(Lg))
    h = ctx.conv(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda(), plan=p).cpu().numpy()
    assert oracle.rel_l2(h, oracle.conv(f, g)) < 1e-11


# ---------------------------------------------------------------- documented search space
def _space(Lout, ndim, axis, N, eb):
    """include/hdconv.h hd_tune's per-axis space restated from its documentation."""
    def r(n):
        k = 128 // eb * 8
        return -(-n // k) * k
    def smem(q, C, D, m, nbuf):
        return eb * (r(q) + r(256) + nbuf * r(C * D * m))
    def default_threads(C, D, m):
        items = C * D * (m // 8)
        best, beff = 576, 0.0
        for nt in range(576, 127, -32):
            eff = items / (-(-items // nt) * nt)
            if eff > beff + 0.01:
                beff, best = eff, nt
        return best
    nbuf = (2 if N == 1 else 3) if axis == 0 else 1
    out = []
    m = 16
    while m <= 4096:
        q = -(-Lout // m)
        if q <= 1024:
            Ds, D = [], q
            while True:
                Ds.append(D)
                if D == 1:
                    break
                D = (D + 1) // 2
            for C in (1, 2, 4, 8):
                for D in Ds:
                    sm = smem(q, C, D, m, nbuf)
                    if sm > 227 * 1024:
                        continue
                    dt = default_threads(C, D, m)
                    ths = [0, dt] + ([256] if dt != 256 else [])
                    if C * D * (m // 8) >= 512 and sm > 227 * 1024 // 2:
                        ths += [t for t in (768, 1024) if t != dt]
                    for S in ((1,) if ndim == 1 else (1, 2, 4, 8, 16)):
                        for th in ths:
                            out.append((m, C, S, D, th))
        m *= 2
    return out


@pytest.mark.parametrize("Lf,Lg,N,c128", [([4096, 4096], [255, 255], 1, True), ([2048, 2048], [1024, 1536], 6, True),
                                          ([8192], [3000], 1, True), ([512, 512, 512], [129, 129, 129], 1, False)])
def test_tune_space_matches_documentation(H, Lf, Lg, N, c128):
    """hd_tune_space (the candidates hd_tune times) equals the space include/hdconv.h
    documents (every power-of-two m that fits shared memory, D in
    {q, ceil(q/2), ..., 1}, C <= 8, S <= 16)."""
    dt = H.HD_C128 if c128 else H.HD_C64
    for ax in range(len(Lf)):
        got = H.tune_space(dt, Lf, Lg, ax, N=N)
        ref = _space(Lf[ax] + Lg[ax] - 1, len(Lf), ax, N, 16 if c128 else 8)
        assert got == ref, (ax, len(got), len(ref))
        assert {c[0] for c in got} >= {512, 1024, 2048}
        assert max(c[2] for c in got) == (16 if len(Lf) > 1 else 1)


@pytest.mark.gpu
def test_per_axis_log_size_is_the_space(ctx, H):
    """Per-axis search (fake costs): one log entry for the starting plan plus one per
    candidate of every axis; exhaustive: the cross product."""
    Lf, Lg = [40, 30], [5, 6]
    ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="per_axis", fake_cost=1, seed=3)
    n0, n1 = (len(H.tune_space(H.HD_C128, Lf, Lg, a)) for a in (0, 1))
    assert len(ctx.hd_tune_log()) == 1 + n0 + n1
    ctx.hd_tune_ex(H.HD_C128, Lf, Lg, mode="exhaustive", fake_cost=1, seed=3)
    assert len(ctx.hd_tune_log()) == n0 * n1
