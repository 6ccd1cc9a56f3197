"""Pins for the oracle's complex-image accumulation mode (beyond the
paper; oracle/ozfft_oracle.c orc_split_shared / orc_execute_image).

* the ring maps a + i b -> a +- iota b (iota^2 = -1 mod p) are homomorphisms Z[i] -> Z_p;
* integer core: the Re / Im CRT integers of every Alg.8 group equal a brute-force COMPLEX
  integer cyclic convolution of the complex digit vectors (definition), so the image
  convolutions, their recombination (z+ + z-)/2, (z+ - z-)/(2 iota) and Garner are exact;
* shared-exponent split: both parts of each level carry the same exponent, digits are
  bounded by 2^alpha and reconstruct x' (hi + lo) exactly up to the final residual;
* alpha: the bound 2 L n 4^alpha < P/2 (a real output sums L n complex products);
* counts: 12 forward + 20 inverse runtime NTTs at (K, L) = (3, 3) without gaps;
* end to end: __float128 direct DFT within the paper's error band.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import workloads


def test_iota_and_homomorphism():
    rng = np.random.default_rng(0)
    for p in (O.P0, O.P1):
        io = O.root_of_unity(p, 4)
        assert io * io % p == p - 1
        for _ in range(50):
            ar, ai, br, bi = (int(v) for v in rng.integers(-2**24, 2**24, 4))
            cr, ci = ar * br - ai * bi, ar * bi + ai * br  # (a)(b) in Z[i]
            for sgn in (1, -1):
                img = lambda r, i: (r + sgn * io * i) % p  # noqa: E731
                assert img(ar, ai) * img(br, bi) % p == img(cr, ci)


def brute_complex_groups(t, wdig, n, m, K, L):
    """Per group: sum_(s,t) sum_{i<n} D_s(i) Dw_t((j-i) mod m) in Z[i], for j < n."""
    out = {}
    j = np.arange(n)
    for g, (cexp, pairs) in enumerate(O.parse_sched(t["sched"][0], L)):
        re = np.zeros(n, dtype=object)
        im = np.zeros(n, dtype=object)
        for s, tt in pairs:
            Dr, Di = t["digits"][0, s].astype(object), t["digits"][1, s].astype(object)
            Wr, Wi = wdig[0, tt].astype(object), wdig[1, tt].astype(object)
            for i in range(n):
                if Dr[i] or Di[i]:
                    wr, wi = Wr[(j - i) % m], Wi[(j - i) % m]
                    re += Dr[i] * wr - Di[i] * wi
                    im += Dr[i] * wi + Di[i] * wr
        out[g] = (re, im)
    return out


@pytest.mark.parametrize("n,dist,seed,cyclic", [(1, "uniform", 0, False), (2, "normal", 1, False),
                                                (7, "signexp", 2, False), (48, "normal", 3, False),
                                                (100, "uniform", 4, False), (64, "signexp", 5, True)])
def test_image_integer_core_bruteforce(n, dist, seed, cyclic):
    K, L = 3, 3
    pl = O.Plan(n, K, L, image=True, cyclic=cyclic)
    x = workloads.draw(dist, seed, 1, n)[0]
    _, t = pl.execute(x, taps=True)
    ref = brute_complex_groups(t, pl.tables()["wdig"], n, pl.m, K, L)
    bound = 2 * L * n * 4 ** pl.alpha
    assert 2 * bound < O.P0 * O.P1
    for g, (re, im) in ref.items():
        assert [int(v) for v in t["crt"][0, g]] == list(re), g
        assert [int(v) for v in t["crt"][1, g]] == list(im), g
        assert max(abs(int(v)) for v in list(re) + list(im) + [0]) <= bound
    assert t["flags"][0] == 0


@pytest.mark.parametrize("n", [3, 100, 1024])
def test_shared_split(n):
    pl = O.Plan(n, 3, 3, image=True)
    x = workloads.phi_input(n, 1.0, seed=n, batch=1)[0]
    _, t = pl.execute(x, taps=True)
    k = int(t["kv"][0])
    assert t["kv"][1] == k and np.array_equal(t["E"][0], t["E"][1])
    a = pl.alpha
    assert np.all(np.abs(t["digits"]) <= 2 ** a)
    # sum_k D_k 2^(E_k - alpha) reproduces x' up to the last level's rounding unit
    xdd = t["xdd"]
    for part in range(2):
        hi, lo = xdd[2 * part], xdd[2 * part + 1]
        for j in range(0, n, max(1, n // 16)):
            rec = sum(Fraction(int(t["digits"][part, kk, j])) * Fraction(2) ** (int(t["E"][part, kk]) - a)
                      for kk in range(k))
            exact = Fraction(float(hi[j])) + Fraction(float(lo[j]))
            assert abs(rec - exact) <= Fraction(2) ** (int(t["E"][part, k - 1]) - a)


@pytest.mark.parametrize("n,L", [(1000, 3), (1 << 18, 3), (1 << 17, 1), (100003, 3)])
def test_image_alpha(n, L):
    """The image plan's alpha is the largest a with 2 L n 4^a < P/2 (bound on a real
    output: L n complex digit products, each |Re| <= 2 4^a)."""
    al = O.Plan(n, 3, L, image=True, cyclic=(n & (n - 1) == 0)).alpha
    P = O.P0 * O.P1
    assert 2 * (2 * L * n * 4 ** al) < P <= 2 * (2 * L * n * 4 ** (al + 1))
    if n == 1 << 18 and L == 3:
        assert al == 20  # = the real-mode L = 3 table entry at log2(2n) = 19


@pytest.mark.parametrize("n", [256, 1024])
def test_image_counts(n):
    pl = O.Plan(n, 3, 3, image=True)
    x = workloads.phi_input(n, 0.0, seed=1, batch=1)[0]
    _, t = pl.execute(x, taps=True)
    assert list(t["counts"]) == [12, 20, 12]  # 32 runtime NTTs vs 52 for the real mode


@pytest.mark.parametrize("n", [1, 16, 37, 1000, 4096])
@pytest.mark.parametrize("dist", ["uniform", "normal", "signexp"])
def test_image_against_float128(n, dist):
    x = workloads.draw(dist, n + 5, 1, n)[0]
    y = O.Plan(n, image=True).execute(x)
    hi, lo = O.dft_f128(x)
    ref = hi + lo
    err = np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-300)
    assert err <= 4e-16, err  # measured <= 1.64e-16 (as tests/test_oracle_pipeline.py PIN)


def test_image_roundtrip_and_nonfinite():
    n = 500
    pl = O.Plan(n, image=True)
    x = workloads.draw("normal", 9, 1, n)[0]
    xr = pl.execute(pl.execute(x), inverse=True)
    assert np.max(np.abs(xr - x)) / np.max(np.abs(x)) <= 1e-15
    x[3] = np.inf
    assert np.all(np.isnan(pl.execute(x)))
