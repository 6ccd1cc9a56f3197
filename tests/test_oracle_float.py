"""Pins for the oracle's float stages: chirp (O1), DD premultiply (O3), Ozaki split (O4).

Each check is against something other than the oracle: mpmath at 200 bits, exact
rational arithmetic (fractions.Fraction), closed forms, and the paper's stated
invariants (eq:ozaki-scheme-split-condition P:359-363, eq:k-upper-limit P:393-399).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import workloads


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 37, 1000, 1024])
def test_chirp_correctly_rounded(n):
    """omega(j) = omega_{2n}^{j^2} -> correctly rounded fp64 (ruling 3)."""
    import mpmath
    mpmath.mp.prec = 200
    Cc, S = O.chirp(n)
    for j in range(n):
        r = (j * j) % (2 * n)
        t = mpmath.mpf(r) / n  # cospi/sinpi are exact at half-integers
        c, s = float(mpmath.cospi(t)), float(-mpmath.sinpi(t))
        if c == 0.0:
            c = 0.0
        if s == 0.0:
            s = 0.0
        # exact zeros at r in {0, n/2, n, 3n/2} are stored as +0.0
        assert (Cc[j], S[j]) == (c, s), (n, j)
        if 2 * r % n == 0:
            assert np.signbit(Cc[j]) == (Cc[j] < 0) and np.signbit(S[j]) == (S[j] < 0)


def test_chirp_closed_forms():
    n = 64
    Cc, S = O.chirp(n)
    j2 = np.arange(n) ** 2 % (2 * n)
    assert np.all(Cc[j2 == 0] == 1.0) and np.all(S[j2 == 0] == 0.0)
    assert np.all(S[j2 == n // 2] == -1.0) and np.all(Cc[j2 == n] == -1.0)


def _fr(v):
    return Fraction(float(v))


def test_premul_dd_error_bound():
    """x' = x (.) omega in DD (Alg.4 step 2): each component within
    2^-104 * (|a b| + |c d|) of the exact value (DD bound, Hida 2001 cited at P:416)."""
    n = 257
    x = workloads.draw("signexp", 11, 1, n)[0]
    Cc, S = O.chirp(n)
    hr, lr, hi, li = O.premul(x, Cc, S)
    for j in range(n):
        xr, xi, c, s = map(_fr, (x[j].real, x[j].imag, Cc[j], S[j]))
        ex_re, ex_im = xr * c - xi * s, xr * s + xi * c
        b_re = (abs(xr * c) + abs(xi * s)) * Fraction(1, 2 ** 104)
        b_im = (abs(xr * s) + abs(xi * c)) * Fraction(1, 2 ** 104)
        assert abs(_fr(hr[j]) + _fr(lr[j]) - ex_re) <= b_re
        assert abs(_fr(hi[j]) + _fr(li[j]) - ex_im) <= b_im
        # DD normalisation: hi = RN(hi + lo)
        assert float(hr[j] + lr[j]) == hr[j] and float(hi[j] + li[j]) == hi[j]
    # conjugate-on-load (inverse wrapper, O10) negates x_im exactly
    hr2, lr2, hi2, li2 = O.premul(np.conj(x), Cc, S)
    hr3, lr3, hi3, li3 = O.premul(x, Cc, S, conj=True)
    assert all(np.array_equal(a, b) for a, b in zip((hr2, lr2, hi2, li2), (hr3, lr3, hi3, li3)))


def _check_split(hi0, lo0, alpha, K):
    k, dig, E, hi, lo = O.split(hi0, lo0, alpha, K)
    assert 0 <= k <= K
    n = hi0.size
    for lvl in range(k):
        assert np.max(np.abs(dig[lvl].astype(np.int64))) <= 2 ** alpha
        if lvl + 1 < k:
            # residual shrinks by ~alpha bits per level (|r| <= 2^(E-alpha), plus one
            # binade for the FastTwoSum rounding of r + lo)
            assert E[lvl + 1] <= E[lvl] - alpha + 1
    # exact reconstruction: sum_k D_k 2^-(alpha-E_k) + hi + lo == x'  (Alg.3 Ensure)
    for j in range(0, n, max(1, n // 97)):
        tot = Fraction(0)
        for lvl in range(k):
            tot += Fraction(int(dig[lvl, j])) * Fraction(2) ** (int(E[lvl]) - alpha)
        tot += _fr(hi[j]) + _fr(lo[j])
        assert tot == _fr(hi0[j]) + _fr(lo0[j])
    return k, dig, E, hi, lo


@pytest.mark.parametrize("dist,seed", [("uniform", 0), ("normal", 1), ("signexp", 3)])
def test_split_invariants(dist, seed):
    n = 1000
    x = workloads.draw(dist, seed, 1, n)[0]
    Cc, S = O.chirp(n)
    hr, lr, hi, li = O.premul(x, Cc, S)
    a = O.alpha(n, 3)
    for h, l in ((hr, lr), (hi, li)):
        k, dig, E, _, _ = _check_split(h, l, a, 3)
        assert k == 3
        # digit grid: c^(k) x^(k) in Z -- the top digit reaches 2^(alpha-1)..2^alpha
        assert 2 ** (a - 1) <= np.max(np.abs(dig[0].astype(np.int64))) <= 2 ** a


def test_split_special_cases():
    a = 22
    z = np.zeros(64)
    k, *_ = _check_split(z, z, a, 3)
    assert k == 0
    imp = np.zeros(64)
    imp[5] = 1.0
    k, dig, E, hi, lo = _check_split(imp, np.zeros(64), a, 3)
    assert k == 1 and dig[0, 5] == 2 ** a and E[0] == 0
    rng = np.random.default_rng(0)
    v = rng.choice([-1.0, 1.0], 64) * 2.0 ** -7  # +-2^e, common exponent
    k, *_ = _check_split(v, np.zeros(64), a, 3)
    assert k == 1


@pytest.mark.parametrize("seed", range(6))
def test_split_count_bound(seed):
    """With no cap, k <= ceil((log2 max - log2 min + log2 u^-1 - 1)/(alpha - 1))
    (eq:k-upper-limit) for fp64 vectors (lo = 0, u = 2^-53)."""
    rng = np.random.default_rng(seed)
    n = 128
    x = (rng.random(n) - 0.5) * np.exp(4.0 * rng.standard_normal(n))  # phi = 4
    x[x == 0] = 1e-3
    a = O.alpha(n, 1)
    k, *_ = _check_split(x, np.zeros(n), a, 8)
    mx, mn = np.max(np.abs(x)), np.min(np.abs(x))
    bound = int(np.ceil((np.log2(mx) - np.log2(mn) + 53 - 1) / (a - 1)))
    assert k <= bound
    if k < 8:
        pass  # exhausted: reconstruction above is then exact with hi = lo = 0
