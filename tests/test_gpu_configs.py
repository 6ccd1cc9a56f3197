"""GPU parity at BASELINE.json's full configurations, in the launch configuration
bench.py times (default plan: K=3, L=3, paper primes, one execute per batch).

The oracle recomputes a seeded sample of transforms one by one: transforms {0, B-1}
plus 6 random ones (all transforms when B <= 8), compared bit-exactly on the fp64
output and, through the taps entry point, on digits, slice counts and CRT integers.
"""
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


def sample(B, seed=0):
    if B <= 8:
        return list(range(B))
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, B - 1), 6, replace=False)
    return sorted({0, B - 1, *[int(v) for v in mid]})


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_forward(oz, name):
    cfg = workloads.CONFIGS[name]
    x = workloads.config_input(cfg)
    plan = oz.Plan(cfg.n, cfg.batch)
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt).cpu().numpy()
    st = plan.stats()
    assert st["nonfinite"] == 0
    op = O.Plan(cfg.n)
    idx = sample(cfg.batch)
    ys, _ = op.execute_batch(np.ascontiguousarray(x[idx]))
    for i, b in enumerate(idx):
        assert np.array_equal(y[b], ys[i]), (name, b)
    # integer stages on the sampled transforms
    if plan.chunk == plan.batch:
        yt, gt = plan.execute_taps(xt)
        assert np.array_equal(yt.cpu().numpy(), y)
        for b in idx[:3]:
            _, ot = op.execute(x[b], taps=True)
            assert np.array_equal(gt["kv"][b].cpu().numpy(), ot["kv"])
            assert np.array_equal(gt["digits"][b].cpu().numpy(), ot["digits"])
            assert np.array_equal(gt["sched"][b].cpu().numpy(), ot["sched"])
            for cv in range(4):
                ng = int(ot["sched"][cv, 0])
                assert np.array_equal(gt["crt"][b, cv, :ng].cpu().numpy(), ot["crt"][cv, :ng])
                assert np.array_equal(gt["res"][b, cv, :ng].cpu().numpy().astype(np.uint32),
                                      ot["res"][cv, :ng])
        # (K,L)=(3,3) on these inputs: 12 forward + 40 inverse NTTs per transform
        assert st["fwd_ntts"] == 12 * cfg.batch and st["inv_ntts"] == 40 * cfg.batch


def test_config_c5_roundtrip(oz):
    cfg = workloads.CONFIGS["c5"]
    x = workloads.config_input(cfg)
    plan = oz.Plan(cfg.n, cfg.batch)
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt)
    xr = plan.inverse(y).cpu().numpy()
    yn = y.cpu().numpy()
    op = O.Plan(cfg.n)
    idx = sample(cfg.batch, seed=4)
    ys, _ = op.execute_batch(np.ascontiguousarray(x[idx]))
    xs, _ = op.execute_batch(np.ascontiguousarray(yn[idx]), inverse=True)
    for i, b in enumerate(idx):
        assert np.array_equal(yn[b], ys[i])
        assert np.array_equal(xr[b], xs[i])
    err = np.max(np.abs(xr - x)) / np.max(np.abs(x))
    assert err <= 1e-15, err


@pytest.mark.parametrize("n,B", [(20000, 3), (300000, 1)])
def test_decomposition_sizes(oz, n, B):
    """NTT decompositions not covered by c1-c5: m = 2^16 (R = 32) and the largest supported
    m = 2^20 (C = 2^12, R = 2^8)."""
    x = workloads.draw("normal", n, B, n)
    plan = oz.Plan(n, B)
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    op = O.Plan(n)
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        assert np.array_equal(y[b].cpu().numpy(), yo)
        assert np.array_equal(gt["digits"][b].cpu().numpy(), ot["digits"])
        for cv in range(4):
            ng = int(ot["sched"][cv, 0])
            assert np.array_equal(gt["crt"][b, cv, :ng].cpu().numpy(), ot["crt"][cv, :ng])


@pytest.mark.parametrize("n,conv", [(600000, "padded"), (1 << 21, "padded"), (1 << 21, "cyclic")])
def test_largest_sizes(oz, n, conv):
    """The largest decompositions this build supports: m = 2^21 (R = 2^9, 32 elements per
    thread in the column passes) and m = 2^22 = 2^10 x 2^12; cyclic m = n = 2^21.  One
    transform, fp64 output bitwise equal to the oracle (whose integer stages are pinned)."""
    x = workloads.draw("uniform", 21, 1, n)
    plan = oz.Plan(n, 1, conv=conv)
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    assert plan.stats()["nonfinite"] == 0
    yo = O.Plan(n, cyclic=(conv == "cyclic")).execute(x[0])
    assert np.array_equal(y[0], yo)
