"""Pins for the oracle's cyclic Bluestein mode.

For a power-of-two n the paper keeps the convolution length N = n: omega*(j) =
omega_2n^{-j^2} has period n for even n, so the Bluestein convolution (eq:bluestein_convolution,
P:183-187) is already cyclic of length n.  The pins:

* integer core: the CRT integers equal a brute-force integer CYCLIC convolution of length n
  of the digit vectors summed per Alg.8 group (definition of cyclic convolution);
* periodicity: the omega~* digits of the cyclic plan are the first n digits of the padded
  plan's (same values, same per-level maxima), and the CRT integers and fp64 outputs of
  the two plans are identical -- the mathematical content of P:238-241;
* end to end: __float128 direct DFT within the paper's error band.
"""
import numpy as np
import pytest

import oracle as O
import workloads

from test_oracle_pipeline import brute_group_ints


@pytest.mark.parametrize("n,dist,seed", [(1, "uniform", 0), (2, "normal", 1), (4, "uniform", 2),
                                         (16, "signexp", 3), (64, "normal", 4),
                                         (128, "uniform", 5)])
def test_cyclic_integer_core_bruteforce(n, dist, seed):
    K, L = 3, 3
    pl = O.Plan(n, K, L, cyclic=True)
    assert pl.m == n
    x = workloads.draw(dist, seed, 1, n)[0]
    _, t = pl.execute(x, taps=True)
    ref = brute_group_ints(t, pl.tables(), n, n, K, L)
    for (cv, g), acc in ref.items():
        assert [int(v) for v in t["crt"][cv, g]] == list(acc), (cv, g)


@pytest.mark.parametrize("n", [2, 8, 256, 1024, 4096])
@pytest.mark.parametrize("dist", ["uniform", "normal", "signexp"])
def test_cyclic_equals_padded(n, dist):
    pc = O.Plan(n, cyclic=True)
    pp = O.Plan(n)
    assert pc.m == n and pp.m == 2 * n and pc.alpha == pp.alpha
    tc, tp = pc.tables(), pp.tables()
    assert np.array_equal(tc["kw"], tp["kw"]) and np.array_equal(tc["Ew"], tp["Ew"])
    assert np.array_equal(tc["wdig"], tp["wdig"][:, :, :n])
    x = workloads.draw(dist, n, 2, n)
    for b in range(2):
        yc, t1 = pc.execute(x[b], taps=True)
        yp, t2 = pp.execute(x[b], taps=True)
        assert np.array_equal(t1["crt"], t2["crt"])
        assert np.array_equal(t1["sched"], t2["sched"])
        assert np.array_equal(yc.view(np.uint64), yp.view(np.uint64))


@pytest.mark.parametrize("n", [1, 4, 64, 1024])
def test_cyclic_against_float128(n):
    x = workloads.draw("uniform", 7, 1, n)[0]
    y = O.Plan(n, cyclic=True).execute(x)
    hi, lo = O.dft_f128(x)
    ref = hi + lo
    err = np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-300)
    assert err <= 4e-16, err  # measured <= 1.64e-16 (as tests/test_oracle_pipeline.py PIN)


def test_cyclic_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        O.Plan(100, cyclic=True)
