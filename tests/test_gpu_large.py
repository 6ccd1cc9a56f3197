"""The full length range of the paper's primes (two-adicity 24 of p0): NTT
lengths m = 2^23 and 2^24 (n <= 2^23), with columns of R = 2^11 / 2^12 rows.

* n = 2^21 + 1 (m = 2^23): output and CRT integers bit-exact against the oracle.
* n = 2^23 (m = 2^24, the limit): the oracle would take minutes, so the pins are the paper's
  own identity P:238-241 -- the padded plan (m = 2^24, R = 2^12) and the N = n cyclic plan
  (m = 2^23, R = 2^11, itself pinned by the first test's decomposition) give bitwise-equal
  spectra --, the __float128 DFT on sampled bins and the round trip.
* beyond the limit: n = 2^23 + 1 is refused (UNSUPPORTED_LENGTH)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    oz.load_library()
    return oz


def test_m_2p23_bit_exact(oz):
    n = (1 << 21) + 1
    x = workloads.draw("normal", 23, 1, n)
    plan = oz.Plan(n, 1)
    assert plan.m == 1 << 23 and plan.log2_rows == 11
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt)
    yo = O.Plan(n).execute(x[0])
    assert np.array_equal(y[0].cpu().numpy(), yo)


def test_m_2p24_limit(oz):
    n = 1 << 23
    x = workloads.draw("uniform", 24, 1, n)
    xt = torch.from_numpy(x).cuda()
    pad = oz.Plan(n, 1)
    assert pad.m == 1 << 24 and pad.log2_rows == 12 and pad.log2_cols == 12
    y = pad.forward(xt)
    cyc = oz.Plan(n, 1, conv="cyclic")
    assert cyc.m == 1 << 23 and cyc.log2_rows == 11
    assert torch.equal(cyc.forward(xt), y)  # same integers, same bits
    del cyc
    yn = y[0].cpu().numpy()
    bins = np.array([0, 1, 12345, n // 2, n - 1, 7654321], dtype=np.int64)
    hi, lo = O.dft_f128(x[0], bins=bins)
    err = np.max(np.abs((yn[bins] - hi) - lo)) / np.max(np.abs(yn))
    assert err <= 1e-15, err
    xr = pad.inverse(y)[0].cpu().numpy()
    assert np.max(np.abs(xr - x[0])) / np.max(np.abs(x[0])) <= 1e-15


def test_beyond_the_primes(oz):
    with pytest.raises(oz.OzfftError) as e:
        oz.Plan((1 << 23) + 1, 1)
    assert e.value.status == 2
