"""Pins for the whole oracle pipeline (O6-O10) and its integer core.

* integer core: the CRT integers equal a brute-force integer cyclic convolution of
  the digit vectors summed over each Alg.8 group;
* transform counts: 52 runtime / 64 total at (K,L)=(3,3), 96 at (3,1)
   and the count laws;
* end to end: __float128 direct DFT (eq:dft P:152-156), closed forms, Parseval,
  linearity and the round trip, within the paper's error band.
"""
import numpy as np
import pytest

import oracle as O
import workloads


def brute_group_ints(taps, tables, n, m, K, L):
    """sum_{(s,t) in g} sum_{i<n} D_{a,s}(i) Dw_{b,t}((j-i) mod m) for j < n, exact ints."""
    conv_ab = [(0, 0), (1, 1), (1, 0), (0, 1)]
    out = {}
    j = np.arange(n)
    for cv, (a, b) in enumerate(conv_ab):
        for g, (cexp, pairs) in enumerate(O.parse_sched(taps["sched"][cv], L)):
            acc = np.zeros(n, dtype=object)
            for s, t in pairs:
                D = taps["digits"][a, s].astype(object)
                Dw = tables["wdig"][b, t].astype(object)
                for i in range(n):
                    if D[i]:
                        acc += D[i] * Dw[(j - i) % m]
            out[(cv, g)] = acc
    return out


@pytest.mark.parametrize("n,dist,seed", [(1, "uniform", 0), (2, "normal", 1), (5, "uniform", 2),
                                         (37, "signexp", 3), (64, "normal", 4),
                                         (100, "uniform", 5)])
def test_integer_core_bruteforce(n, dist, seed):
    K, L = 3, 3
    pl = O.Plan(n, K, L)
    x = workloads.draw(dist, seed, 1, n)[0]
    y, t = pl.execute(x, taps=True)
    tab = pl.tables()
    ref = brute_group_ints(t, tab, n, pl.m, K, L)
    bound = L * n * 4 ** pl.alpha
    assert 2 * bound < O.P0 * O.P1  # the alpha condition
    for (cv, g), acc in ref.items():
        got = t["crt"][cv, g]
        assert [int(v) for v in got] == list(acc), (cv, g)
        assert np.max(np.abs(got)) <= bound
    assert t["flags"][0] == 0


def test_schedule_no_gap_groups():
    """No gaps: groups are the anti-diagonals, at most L per group (Alg.8)."""
    a = 20
    sx = [a - 0, a + a, a + 2 * a]  # s_k = alpha - E_k with E_k = -k alpha
    sw = list(sx)
    groups, _ = O.schedule(sx, sw, 3, 3)
    assert [pairs for _, pairs in groups] == [
        [(2, 2)], [(1, 2), (2, 1)], [(0, 2), (1, 1), (2, 0)], [(0, 1), (1, 0)], [(0, 0)]]
    assert [c for c, _ in groups] == [sx[2] + sw[2], sx[1] + sw[2], sx[0] + sw[2],
                                      sx[0] + sw[1], sx[0] + sw[0]]
    # L = 1: every pair its own group, 2 K^2 inverse NTTs per real conv
    groups1, _ = O.schedule(sx, sw, 3, 1)
    assert len(groups1) == 9
    # L = 2 splits the middle anti-diagonal (l >= L flush, line 972)
    groups2, _ = O.schedule(sx, sw, 3, 2)
    assert [pairs for _, pairs in groups2] == [
        [(2, 2)], [(1, 2), (2, 1)], [(0, 2), (1, 1)], [(2, 0)], [(0, 1), (1, 0)], [(0, 0)]]
    # a gap breaks the equal-scale chain (c differs -> flush)
    sx_gap = [a, 2 * a + 3, 3 * a + 3]
    gg, _ = O.schedule(sx_gap, sw, 3, 3)
    for c, pairs in gg:
        assert len({sx_gap[s] + sw[t] for s, t in pairs}) == 1 and c == sx_gap[pairs[0][0]] + sw[pairs[0][1]]
    assert sum(len(p) for _, p in gg) == 9
    assert O.schedule([], sw, 3, 3)[0] == []


@pytest.mark.parametrize("n", [256, 1024])
def test_transform_counts_paper(golden, n):
    g = golden["ntt_counts"]
    x = workloads.phi_input(n, 0.0, seed=n, batch=1)[0]  # phi = 0
    _, t = O.Plan(n, 3, 3).execute(x, taps=True)
    fwd, inv, cached = (int(v) for v in t["counts"])
    assert fwd + inv == g["K3_L3_runtime"]          # 52
    assert fwd + inv + cached == g["K3_L3_total"]   # 64
    assert fwd + inv + cached == 24 * 3 - 8         # 24K - 8
    _, t1 = O.Plan(n, 3, 1).execute(x, taps=True)
    assert int(t1["counts"].sum()) == g["K3_L1_total"]  # 96
    assert int(t1["counts"][:2].sum()) == 4 * 3 + 8 * 9  # 4K + 8K^2


def rel_err(y, hi, lo):
    return np.max(np.abs((y - hi) - lo)) / np.max(np.abs(hi))


# The oracle's measured error against the __float128 DFT is <= 1.64e-16 relative to norm over
# every case below (padded, cyclic, image and TS modes alike; dominated by the fp64 chirp
# rounding).  The pin is 4e-16, well inside the paper's [1e-16, 1e-15] band, so
# a slip in the DD recombination or post-chirp (a dropped low word, a wrong flush order)
# that costs a few ulps shows up here.
PIN = 4e-16


@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 37, 64, 100, 256, 997, 1024])
@pytest.mark.parametrize("dist", ["uniform", "normal", "signexp"])
def test_against_float128_dft(golden, n, dist):
    x = workloads.draw(dist, n, 1, n)[0]
    y = O.Plan(n).execute(x)
    hi, lo = O.dft_f128(x)
    e = rel_err(y, hi, lo)
    assert e <= PIN, e
    assert e <= golden["error_band"]["hi"]


def test_against_float128_bins_large():
    n = 1 << 12
    x = workloads.draw("uniform", 9, 1, n)[0]
    y = O.Plan(n).execute(x)
    bins = np.random.default_rng(0).choice(n, 64, replace=False)
    hi, lo = O.dft_f128(x, bins=bins)
    full_hi, _ = O.dft_f128(x, bins=None) if n <= 4096 else (None, None)
    assert np.max(np.abs((y[bins] - hi) - lo)) / np.max(np.abs(full_hi)) <= PIN


@pytest.mark.parametrize("n", [8, 13, 64, 100])
def test_closed_forms(n):
    pl = O.Plan(n)
    k = np.arange(n)
    tol = 1e-15
    imp = np.zeros(n, np.complex128)
    imp[0] = 1
    assert np.max(np.abs(pl.execute(imp) - 1)) <= tol  # impulse -> ones
    j0 = 3 % n
    imp = np.zeros(n, np.complex128)
    imp[j0] = 1
    ref = np.exp(-2j * np.pi * ((j0 * k) % n) / n)  # omega_n^{j0 k}
    assert np.max(np.abs(pl.execute(imp) - ref)) <= 2 * tol
    c = 0.75 - 0.25j
    y = pl.execute(np.full(n, c))
    assert abs(y[0] - n * c) <= tol * n and np.max(np.abs(y[1:])) <= tol * n
    f = 5 % n
    tone = np.exp(2j * np.pi * ((f * k) % n) / n)
    y = pl.execute(tone)
    ref = np.zeros(n, np.complex128)
    ref[f] = n
    assert np.max(np.abs(y - ref)) <= 4 * tol * n


def test_parseval_linearity_roundtrip():
    n = 1000
    pl = O.Plan(n)
    x = workloads.draw("normal", 1, 1, n)[0]
    z = workloads.draw("uniform", 2, 1, n)[0]
    y = pl.execute(x)
    assert abs(np.sum(np.abs(y) ** 2) - n * np.sum(np.abs(x) ** 2)) <= 1e-14 * n * np.sum(np.abs(x) ** 2)
    a, b = 0.5, -2.0
    yl = pl.execute(a * x + b * z)
    assert np.max(np.abs(yl - (a * y + b * pl.execute(z)))) <= 1e-15 * np.max(np.abs(yl)) * 4
    xr = pl.execute(y, inverse=True)
    assert np.max(np.abs(xr - x)) / np.max(np.abs(x)) <= 1e-15
    hi, lo = O.dft_f128(y, inverse=True)
    assert rel_err(xr, hi, lo) <= PIN


def test_nonfinite_and_zero():
    n = 50
    pl = O.Plan(n)
    x = workloads.draw("uniform", 3, 1, n)[0]
    x[7] = np.nan
    y, t = pl.execute(x, taps=True)
    assert np.all(np.isnan(y)) and t["flags"][0] & 1
    y, t = pl.execute(np.zeros(n, np.complex128), taps=True)
    assert np.all(y == 0) and int(t["counts"][0] + t["counts"][1]) == 0


def test_batch_matches_single():
    n = 100
    pl = O.Plan(n)
    x = workloads.draw("normal", 4, 6, n)
    yb, used = pl.execute_batch(x)
    assert used >= 1
    for b in range(6):
        assert np.array_equal(yb[b], pl.execute(x[b]))


@pytest.mark.parametrize("n,signs", [(4, "plus"), (64, "plus"), (64, "random"), (1000, "plus"),
                                     (1000, "random")])
def test_integer_core_adversarial_bound(n, signs):
    """digits all at +-2^alpha and groups of L = 3 pairs -- the largest sums the
    alpha condition allows (L n 4^alpha < P/2) -- are still recovered exactly by
    the oracle's NTT-domain accumulation, inverse NTT and Garner."""
    L = 3
    a = O.alpha(n, L)
    m = 1
    while m < 2 * n - 1:
        m <<= 1
    rng = np.random.default_rng(n)
    big = 2 ** a

    def vec(length):
        v = np.full(length, big, dtype=np.int64)
        if signs == "random":
            v *= rng.choice([-1, 1], length)
        return v

    xs = [np.concatenate([vec(n), np.zeros(m - n, np.int64)]) for _ in range(L)]
    ws = [vec(m) for _ in range(L)]
    for w in ws:
        w[n:m - n + 1] = 0  # omega~* support: j < n and j > m - n (ZeroPad_pm)
    exact = np.zeros(n, dtype=object)
    for x, w in zip(xs, ws):
        xo, wo = x.astype(object), w.astype(object)
        for j in range(n):
            exact[j] += sum(xo[i] * wo[(j - i) % m] for i in range(n))
    assert max(abs(int(v)) for v in exact) <= L * n * big * big < O.P0 * O.P1 // 2
    res = []
    for p in (O.P0, O.P1):
        acc = np.zeros(m, dtype=np.uint64)
        for x, w in zip(xs, ws):
            X = O.ntt(np.mod(x, p).astype(np.uint32), p).astype(np.uint64)
            W = O.ntt(np.mod(w, p).astype(np.uint32), p).astype(np.uint64)
            acc = (acc + X * W % p) % p
        res.append(O.ntt(acc.astype(np.uint32), p, inverse=True))
    got = [O.garner2(int(res[0][j]), int(res[1][j]))[0] for j in range(n)]
    assert got == [int(v) for v in exact]
