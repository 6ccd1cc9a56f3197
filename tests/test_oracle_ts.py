"""Pins for the oracle's triple-single (TS) working precision (
P:418-430; Alg.4 TS form; TS split P:784-798).  The paper does not give TSAdd / TSMul;
the oracle's sequences (DESIGN ruling 24) are pinned here against exact rationals:

* TS(double) and TS(int64 < 2^62) are exact, words non-overlapping (|x_s| <= ulp(x_{s-1})/2);
* fl64(TS) is the correctly rounded binary64 of x0 + x1 + x2;
* TSAdd / TSMul: relative error <= 2^-62 (vs |a| + |b| resp. |a b|) on random operands,
  including cancellation-heavy sums; results are non-overlapping triples;
* TS split: |D| <= 2^alpha, every digit an integer, and the digits reconstruct the TS input
  to within the last level's unit 2^(E_last - alpha) (Alg.6 invariant);
* end to end: __float128 direct DFT within the paper's band; the TS pipeline's NTT counts
  obey the same laws as the DD one.
"""
import math
from fractions import Fraction as F

import numpy as np
import pytest

import oracle as O
import workloads


def val(t):
    return F(float(t.x0)) + F(float(t.x1)) + F(float(t.x2))


def ulp32(x):
    x = abs(float(np.float32(x)))
    if x == 0:
        return 0.0
    return float(np.spacing(np.float32(x)))


def nonoverlap(t):
    w = t.words()
    for a, b in ((w[0], w[1]), (w[1], w[2])):
        if a != 0:
            assert abs(b) <= ulp32(a) / 2 * (1 + 1e-9), w


def rand_doubles(rng, k, lo=-60, hi=60):
    return [float(s * m * 2.0 ** e) for s, m, e in zip(rng.choice([-1, 1], k), rng.random(k) + 0.5,
                                                           rng.integers(lo, hi, k))]


def test_ts_conversions_exact():
    rng = np.random.default_rng(1)
    # exact while the third word stays a normal fp32: |d| >= 2^-78 (the TS exponent range is
    # fp32's)
    for d in rand_doubles(rng, 2000, -70, 100) + [0.0, 1.0, -0.1, 2.0 ** -126, 3.0 ** 30]:
        t = O.ts_from_double(d)
        assert val(t) == F(d)
        nonoverlap(t)
        assert O.ts_to_double(t) == d
    for v in [0, 1, -1, 2 ** 40 + 1, -(2 ** 61) + 12345] + [int(x) for x in rng.integers(-2 ** 62, 2 ** 62, 2000, dtype=np.int64)]:
        t = O.ts_from_int64(v)
        assert val(t) == v
        nonoverlap(t)


def test_ts_to_double_correctly_rounded():
    rng = np.random.default_rng(2)
    for _ in range(2000):
        a = O.ts_mul(O.ts_from_double(rand_doubles(rng, 1)[0]), O.ts_from_double(rand_doubles(rng, 1)[0]))
        exact = val(a)
        d = O.ts_to_double(a)
        # no binary64 is closer to the exact value than d
        for nb in (math.nextafter(d, math.inf), math.nextafter(d, -math.inf)):
            assert abs(F(nb) - exact) >= abs(F(d) - exact)


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_ts_add_mul_error_bounds(seed):
    rng = np.random.default_rng(seed)
    bound = F(1, 2 ** 62)
    worst_add = worst_mul = F(0)
    for _ in range(3000):
        a = O.ts_mul(O.ts_from_double(rand_doubles(rng, 1, -20, 20)[0]), O.ts_from_double(rand_doubles(rng, 1, -20, 20)[0]))
        b = O.ts_mul(O.ts_from_double(rand_doubles(rng, 1, -20, 20)[0]), O.ts_from_double(rand_doubles(rng, 1, -20, 20)[0]))
        if rng.random() < 0.3:  # cancellation: b close to -a
            b = O.ts_add(O.ts_mul(a, O.ts_from_double(-1.0)), O.ts_from_double(rand_doubles(rng, 1, -80, -60)[0]))
        s = O.ts_add(a, b)
        nonoverlap(s)
        den = abs(val(a)) + abs(val(b))
        if den:
            worst_add = max(worst_add, abs(val(s) - (val(a) + val(b))) / den)
        p = O.ts_mul(a, b)
        nonoverlap(p)
        ex = val(a) * val(b)
        if ex:
            worst_mul = max(worst_mul, abs(val(p) - ex) / abs(ex))
    assert worst_add <= bound, float(worst_add)
    assert worst_mul <= bound, float(worst_mul)


@pytest.mark.parametrize("alpha,K", [(20, 3), (24, 3), (12, 8)])
def test_ts_split_digits(alpha, K):
    rng = np.random.default_rng(alpha)
    n = 257
    ts = [O.ts_mul(O.ts_from_double(float(v)), O.ts_from_double(1.0 / 3.0))
          for v in rng.standard_normal(n) * np.exp(2 * rng.standard_normal(n))]
    r = np.array([[t.x0 for t in ts], [t.x1 for t in ts], [t.x2 for t in ts]], np.float32)
    orig = [val(t) for t in ts]
    k, dig, E, rr = O.split_ts(r, alpha, K)
    assert 1 <= k <= K
    assert np.all(np.abs(dig[:k]) <= 2 ** alpha)
    for j in range(n):
        rec = sum(F(int(dig[i, j])) * F(2) ** (int(E[i]) - alpha) for i in range(k))
        res = F(float(rr[0, j])) + F(float(rr[1, j])) + F(float(rr[2, j]))
        assert abs(orig[j] - rec) <= F(2) ** (int(E[k - 1]) - alpha + 1)
        if k < K:  # split exhausted: the residual is zero (mu == 0 stopped it)
            assert res == 0


@pytest.mark.parametrize("n", [1, 16, 100, 1024, 4096])
@pytest.mark.parametrize("dist", ["uniform", "normal", "signexp"])
def test_ts_against_float128(n, dist):
    x = workloads.draw(dist, n + 11, 1, n)[0]
    y = O.Plan(n, ts=True).execute(x)
    hi, lo = O.dft_f128(x)
    ref = hi + lo
    err = np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-300)
    assert err <= 4e-16, err  # measured <= 1.64e-16 (as tests/test_oracle_pipeline.py PIN)


def test_ts_counts_and_roundtrip():
    n = 1024
    pl = O.Plan(n, 3, 3, ts=True)
    x = workloads.phi_input(n, 0.0, seed=2, batch=1)[0]
    y, t = pl.execute(x, taps=True)
    c = t["counts"]
    assert c[0] == 2 * int(t["kv"].sum()) and c[1] == 2 * sum(int(t["sched"][cv, 0]) for cv in range(4))
    assert c[0] + c[1] + c[2] == 64  # phi = 0, (K, L) = (3, 3): 24K - 8
    xr = pl.execute(y, inverse=True)
    assert np.max(np.abs(xr - x)) / np.max(np.abs(x)) <= 1e-15
    assert O.Plan(n, ts=True, image=False).alpha == O.Plan(n).alpha
