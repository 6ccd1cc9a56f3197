"""GPU parity of the cyclic Bluestein plans (conv="cyclic", m = n for power-of-two n;
P:238-241) against the oracle's cyclic mode, through the C ABI.

Bar: every integer tap (digits, X, W, Z, residues, CRT integers, schedules) bit-exact
against oracle.Plan(n, cyclic=True); the fp64 output bitwise equal to it AND to the padded
oracle (the two conventions give identical CRT integers, tests/test_oracle_cyclic.py).
Sizes cover the one-pass rows (m <= 4096), two-pass plans with every column length the
decomposition uses, unpruned last column stage (n = m), and BASELINE configs c2/c3/c5
sampled as in tests/test_gpu_configs.py.
"""
import functools

import numpy as np
import pytest
import torch

import oracle as O
import workloads
from test_gpu_configs import sample
from test_gpu_parity import check_taps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    oz.load_library()
    return oz


@functools.lru_cache(maxsize=8)
def oplan(n, cyclic, K=3, L=3):
    return O.Plan(n, K, L, cyclic=cyclic)


@pytest.mark.parametrize("n,B,dist,seed", [
    (1, 1, "uniform", 0), (2, 2, "normal", 1), (16, 2, "signexp", 2), (1024, 2, "uniform", 3),
    (4096, 1, "normal", 4), (1 << 13, 2, "signexp", 5), (1 << 15, 1, "uniform", 6),
    (1 << 16, 1, "normal", 7)])
def test_cyclic_taps_bit_exact(oz, n, B, dist, seed):
    x = workloads.draw(dist, seed, B, n)
    plan = oz.Plan(n, B, conv="cyclic")
    op = oplan(n, True)
    assert plan.m == n == op.m and plan.alpha == op.alpha
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    assert np.array_equal(gt["W"].cpu().numpy().astype(np.uint32), op.tables()["W"])
    yg = y.cpu().numpy()
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        check_taps(gt, ot, n, 3, b)
        assert np.array_equal(yg[b], yo)
        assert np.array_equal(yg[b], oplan(n, False).execute(x[b]))


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_cyclic_configs(oz, name):
    cfg = workloads.CONFIGS[name]
    x = workloads.config_input(cfg)
    xt = torch.from_numpy(x).cuda()
    plan = oz.Plan(cfg.n, cfg.batch, conv="cyclic")
    y = plan.forward(xt)
    yn = y.cpu().numpy()
    idx = sample(cfg.batch, seed=1)
    op = O.Plan(cfg.n)  # padded oracle: identical bits by P:238-241
    ys, _ = op.execute_batch(np.ascontiguousarray(x[idx]))
    for i, b in enumerate(idx):
        assert np.array_equal(yn[b], ys[i]), (name, b)
    st = plan.stats()
    assert st["fwd_ntts"] == 12 * cfg.batch and st["inv_ntts"] == 40 * cfg.batch
    if cfg.roundtrip:
        xr = plan.inverse(y).cpu().numpy()
        xs, _ = op.execute_batch(np.ascontiguousarray(yn[idx]), inverse=True)
        for i, b in enumerate(idx):
            assert np.array_equal(xr[b], xs[i])


def test_cyclic_equals_padded_gpu(oz):
    """Both GPU plans agree bit for bit on a full batch (no oracle sampling)."""
    n, B = 1 << 14, 8
    x = torch.from_numpy(workloads.draw("signexp", 3, B, n)).cuda()
    yc = oz.Plan(n, B, conv="cyclic").forward(x)
    yp = oz.Plan(n, B).forward(x)
    assert torch.equal(yc, yp)


def test_cyclic_rejects_non_power_of_two(oz):
    with pytest.raises(oz.OzfftError):
        oz.Plan(1000, 1, conv="cyclic")
