"""GPU parity of the triple-single plans (precision="ts") against the
oracle's TS mode (oracle.Plan(..., ts=True)), through the C ABI.

Bar: digits, exponents, slice counts, forward spectra, Z, residues, CRT integers and the
schedules bit-exact; fp64 output bitwise equal (same fp32 op sequences on both sides).
Also: the paper's phi = 4 count of 80 NTTs at (K, L) = (3, 3), which the TS split
reproduces (the DD split does not), and the BASELINE configs sampled.
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
def oplan(n, K=3, L=3, cyclic=False):
    return O.Plan(n, K, L, ts=True, cyclic=cyclic)


@pytest.mark.parametrize("n,B,dist,seed", [
    (1, 1, "uniform", 0), (3, 2, "normal", 1), (100, 2, "signexp", 2), (1000, 2, "uniform", 3),
    (2047, 1, "normal", 4), (3001, 2, "signexp", 5), (1 << 13, 2, "normal", 6)])
def test_ts_taps_bit_exact(oz, n, B, dist, seed):
    x = workloads.draw(dist, seed, B, n)
    plan = oz.Plan(n, B, precision="ts")
    op = oplan(n)
    assert plan.m == op.m and plan.alpha == op.alpha and plan.rho == 24 - plan.alpha
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    assert np.array_equal(gt["W"].cpu().numpy().astype(np.uint32), op.tables()["W"])
    yg = y.cpu().numpy()
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        check_taps(gt, ot, n, 3, b)
        assert np.array_equal(yg[b], yo)


@pytest.mark.parametrize("n,phi", [(4096, 4.0), (16384, 4.0), (4096, 0.0)])
def test_ts_phi4_count_80(oz, n, phi):
    """(K, L) = (3, 3): 64 NTT calls at phi = 0, and 80 at phi = 4 with TS splits
    ('For phi = 4.0, the maximum count for (K, L) = (3, 3) was 80')."""
    x = workloads.phi_input(n, phi, seed=n, batch=1)
    plan = oz.Plan(n, 1, precision="ts")
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    st = plan.stats()
    assert st["fwd_ntts"] + st["inv_ntts"] + st["cached_ntts"] == (80 if phi == 4.0 else 64)
    assert np.array_equal(y[0], oplan(n).execute(x[0]))


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_ts_configs(oz, name):
    cfg = workloads.CONFIGS[name]
    x = workloads.config_input(cfg)
    plan = oz.Plan(cfg.n, cfg.batch, precision="ts")
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    idx = sample(cfg.batch, seed=3)[:4]
    ys, _ = oplan(cfg.n).execute_batch(np.ascontiguousarray(x[idx]))
    for i, b in enumerate(idx):
        assert np.array_equal(y[b], ys[i]), (name, b)


def test_ts_inverse_cyclic_and_errors(oz):
    n, B = 1 << 12, 2
    x = workloads.draw("normal", 8, B, n)
    plan = oz.Plan(n, B, precision="ts", conv="cyclic")
    y = plan.forward(torch.from_numpy(x).cuda())
    xr = plan.inverse(y).cpu().numpy()
    yn = y.cpu().numpy()
    op = oplan(n, cyclic=True)
    for b in range(B):
        assert np.array_equal(yn[b], op.execute(x[b]))
        assert np.array_equal(xr[b], op.execute(yn[b], inverse=True))
    hi, lo = O.dft_f128(x[0])
    assert np.max(np.abs((yn[0] - hi) - lo)) / np.max(np.abs(hi)) <= 1e-15
    with pytest.raises(oz.OzfftError):
        oz.Plan(n, 1, precision="ts", accum="image")
