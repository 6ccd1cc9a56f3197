"""Pins for the oracle's integer stages (O0, O5-O8), against what the paper and the
mathematics fix -- never against the oracle itself.

Sources: PAPER.md P:142-149 (symmetric remainder), P:244-313 (NTT, CRT, Garner),
P:720/P:1046 (primes), P:724/P:1178 (alpha values).
"""
import math
import random

import numpy as np
import pytest
import sympy

import oracle as O


# ------------------------------------------------------------------ constants
def test_primes_and_generators(golden):
    p0, p1 = golden["primes"]["p0"], golden["primes"]["p1"]
    assert (O.P0, O.P1) == (p0, p1)
    for p, adic in ((p0, golden["spec_examples"]["two_adicity"]["p0"]),
                    (p1, golden["spec_examples"]["two_adicity"]["p1"])):
        assert sympy.isprime(p)
        assert sympy.multiplicity(2, p - 1) == adic
        # the oracle's primitive root is the smallest one (ruling 4), checked by sympy
        assert O.primitive_root(p) == sympy.primitive_root(p)
        assert p < 2 ** 31 and 2 * p < 2 ** 32
    assert p0 * p1 < 2 ** 62


@pytest.mark.parametrize("p", [O.P0, O.P1])
@pytest.mark.parametrize("logm", [0, 1, 2, 5, 11, 19, 24])
def test_root_of_unity_order(p, logm):
    m = 1 << logm
    w = O.root_of_unity(p, m)
    assert pow(w, m, p) == 1
    if m > 1:
        assert pow(w, m // 2, p) == p - 1  # exact order m


def test_sym_mod_examples(golden):
    for a, m, r in golden["spec_examples"]["sym_mod"]:
        assert O.sym_mod(a, m) == r
    rng = random.Random(5)
    for _ in range(2000):
        m = rng.randrange(1, 10 ** 9)
        a = rng.randrange(-(2 ** 62), 2 ** 62)
        r = O.sym_mod(a, m)
        assert -m / 2 <= r < m / 2 and (a - r) % m == 0


def test_mod_inv_example(golden):
    assert O.lib().orc_invmod(2, O.P0) == golden["spec_examples"]["mod_inv_2_p0"]


# ------------------------------------------------------------------ alpha
def test_alpha_paper_values(golden):
    p0, p1 = golden["primes"]["p0"], golden["primes"]["p1"]
    for c in golden["alpha"]["cases"]:
        assert O.alpha(c["n"], c["L"], p0, p1) == c["alpha"], c


@pytest.mark.parametrize("n", [1, 2, 3, 37, 1000, 1024, 100003, 1 << 14, 1 << 18, 1 << 23])
@pytest.mark.parametrize("L", [1, 2, 3, 4])
def test_alpha_formula_high_precision(n, L):
    """alpha = floor((log2(p0 p1/2) - log2(L n))/2) evaluated with mpmath at
    100 digits -- an independent evaluation of the printed formula."""
    import mpmath
    mpmath.mp.dps = 100
    v = (mpmath.log(mpmath.mpf(O.P0) * O.P1 / 2, 2) - mpmath.log(mpmath.mpf(L) * n, 2)) / 2
    assert O.alpha(n, L) == int(mpmath.floor(v))


def test_alpha_original_ozaki(golden):
    """Fig. 1 fact: the original Ozaki alpha = floor((log2 u^-1 - log2 n)/2) is 2 at
    n = 2^20 in single precision; this pins our reading of the floor."""
    g = golden["alpha_original_ozaki_single_precision"]
    assert math.floor((g["u_log2_inv"] - math.log2(g["n"])) / 2) == g["alpha"]


# ------------------------------------------------------------------ Garner / CRT
def test_garner_examples(golden):
    for z0, z1, v in golden["spec_examples"]["garner2"]:
        assert O.garner2(z0, z1) == (v, False)


def test_garner_exhaustive_small_pair():
    """All (z0, z1) for the test pair (7, 11): unique v in [-P/2, P/2)."""
    p0, p1 = 7, 11
    P = p0 * p1
    seen = set()
    for z0 in range(p0):
        for z1 in range(p1):
            v, fix = O.garner2(z0, z1, p0, p1)
            assert not fix
            assert -P / 2 <= v < P / 2
            assert v % p0 == z0 and v % p1 == z1
            seen.add(v)
    assert len(seen) == P


def test_garner_random_paper_primes():
    rng = random.Random(7)
    P = O.P0 * O.P1
    for _ in range(20000):
        v = rng.randrange(-(P // 2), P // 2 + 1)
        got, fix = O.garner2(v % O.P0, v % O.P1)
        assert got == v and not fix


# ------------------------------------------------------------------ NTT
def ntt_definition(x, p, inverse=False):
    """eq:ntt / eq:intt evaluated literally with Python big ints."""
    m = len(x)
    w = O.root_of_unity(p, m)  # the root is pinned separately above
    if inverse:
        w = pow(w, p - 2, p)
    y = [sum(int(x[j]) * pow(w, j * k, p) for j in range(m)) % p for k in range(m)]
    if inverse:
        minv = pow(m, p - 2, p)
        y = [(v * minv) % p for v in y]
    return y


@pytest.mark.parametrize("p", [O.P0, O.P1])
@pytest.mark.parametrize("m", [1, 2, 4, 8, 32, 64])
def test_ntt_matches_definition(p, m):
    rng = np.random.default_rng(m)
    x = rng.integers(0, p, m, dtype=np.uint64).astype(np.uint32)
    assert list(O.ntt(x, p)) == ntt_definition(x, p)
    assert list(O.ntt(x, p, inverse=True)) == ntt_definition(x, p, inverse=True)


@pytest.mark.parametrize("p", [O.P0, O.P1])
def test_ntt_closed_forms_and_roundtrip(p):
    for m in (1, 2, 16, 1024, 1 << 14):
        imp = np.zeros(m, np.uint32)
        imp[0] = 1
        assert np.all(O.ntt(imp, p) == 1)
        c = 123456789 % p
        y = O.ntt(np.full(m, c, np.uint32), p)
        assert y[0] == (m * c) % p and np.all(y[1:] == 0)
        x = np.random.default_rng(m).integers(0, p, m, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(O.ntt(O.ntt(x, p), p, inverse=True), x)
        assert np.all(O.ntt(np.ones(m, np.uint32), p, inverse=True) == imp)


def test_exact_convolution_via_two_primes(golden):
    """Convolution theorem + Garner reproduce the integer cyclic convolution."""
    def conv(x, y):
        m = len(x)
        xs = [v % O.P0 for v in x], [v % O.P1 for v in x]
        ys = [v % O.P0 for v in y], [v % O.P1 for v in y]
        z = []
        for q, p in enumerate((O.P0, O.P1)):
            X = O.ntt(np.array(xs[q], np.uint32), p)
            Y = O.ntt(np.array(ys[q], np.uint32), p)
            Z = (X.astype(object) * Y.astype(object)) % p
            z.append(O.ntt(np.array(Z, dtype=np.uint64).astype(np.uint32), p, inverse=True))
        return [O.garner2(int(a), int(b))[0] for a, b in zip(*z)]

    assert conv([1, 1, 1, 1], [1, 1, 1, 1]) == golden["spec_examples"]["allones_conv_n4"]
    rng = random.Random(3)
    m = 256
    x = [rng.randint(-(2 ** 20), 2 ** 20) for _ in range(m)]
    y = [rng.randint(-(2 ** 20), 2 ** 20) for _ in range(m)]
    brute = [sum(x[i] * y[(j - i) % m] for i in range(m)) for j in range(m)]
    assert conv(x, y) == brute
    d = [0] * m
    d[0] = 1
    assert conv(d, y) == y
