"""GPU parity of the one-launch small-transform kernel (k_small_fused: one-pass plans,
2^8 <= m <= 2^12, default mode) through the C ABI.

Bar: the fp64 output bitwise equal to the CPU oracle's (forward and inverse, padded and
cyclic plans, ragged / prime n, every input distribution of BASELINE's configs), and
bitwise equal to the three-kernel path of the same plan (OZFFT_SMALL_FUSED=0 at plan
create), whose integer taps tests/test_gpu_parity.py pins stage by stage.  The
per-transform records (slice counts, exponents, schedules -> NTT counts, non-finite flag)
the kernel leaves in the workspace must equal the three-kernel path's.
"""
import functools

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


@functools.lru_cache(maxsize=16)
def oplan(n, cyclic=False, K=3, L=3):
    return O.Plan(n, K, L, cyclic=cyclic)


def plans(oz, monkeypatch, n, B, **kw):
    fused = oz.Plan(n, B, **kw)
    monkeypatch.setenv("OZFFT_SMALL_FUSED", "0")
    multi = oz.Plan(n, B, **kw)
    monkeypatch.delenv("OZFFT_SMALL_FUSED")
    return fused, multi


def launches(oz, fn):
    torch.cuda.synchronize()
    l0 = oz.kernel_launches()
    out = fn()
    torch.cuda.synchronize()
    return out, oz.kernel_launches() - l0


# m = 2^8 .. 2^12: n = 65 .. 2048 (the c1 size n = 2^10 among them), ragged and prime n
@pytest.mark.parametrize("n,B,dist,seed", [
    (65, 2, "uniform", 10), (100, 1, "normal", 11), (128, 3, "signexp", 12),
    (129, 1, "uniform", 13), (500, 2, "normal", 14), (997, 1, "signexp", 15),
    (1000, 2, "uniform", 16), (1024, 1, "uniform", 0), (1025, 1, "normal", 17),
    (1500, 2, "signexp", 18), (2047, 1, "normal", 19), (2048, 2, "uniform", 20),
])
def test_small_fused_bitwise(oz, monkeypatch, n, B, dist, seed):
    x = workloads.draw(dist, seed, B, n)
    xt = torch.from_numpy(x).cuda()
    fused, multi = plans(oz, monkeypatch, n, B)
    assert fused.log2_rows == 0 and 8 <= fused.log2_cols <= 12
    y, nl = launches(oz, lambda: fused.forward(xt))
    assert nl == 1, nl  # ONE launch for the whole path
    ym = multi.forward(xt)
    assert torch.equal(y, ym)
    assert fused.stats() == multi.stats()
    yn = y.cpu().numpy()
    op = oplan(n)
    for b in range(B):
        assert np.array_equal(yn[b], op.execute(x[b])), b
    # inverse direction (conj on load, conj + RN / n at the finish)
    xr = fused.inverse(y)
    assert torch.equal(xr, multi.inverse(ym))
    xo = op.execute(yn[0], inverse=True)
    assert np.array_equal(xr[0].cpu().numpy(), xo)
    assert np.max(np.abs(xr.cpu().numpy() - x)) <= 1e-15 * np.max(np.abs(x))


@pytest.mark.parametrize("n", [256, 1024, 4096])
def test_small_fused_cyclic(oz, monkeypatch, n):
    x = workloads.draw("normal", 30 + n, 2, n)
    xt = torch.from_numpy(x).cuda()
    fused, multi = plans(oz, monkeypatch, n, 2, conv="cyclic")
    assert fused.m == n
    y = fused.forward(xt)
    assert torch.equal(y, multi.forward(xt))
    op = oplan(n, cyclic=True)
    assert np.array_equal(y[1].cpu().numpy(), op.execute(x[1]))


@pytest.mark.parametrize("K,L", [(2, 1), (4, 2), (3, 1)])
def test_small_fused_other_KL(oz, monkeypatch, K, L):
    n = 700
    x = workloads.draw("signexp", 40 + K * 4 + L, 2, n)
    xt = torch.from_numpy(x).cuda()
    fused, multi = plans(oz, monkeypatch, n, 2, K=K, L=L)
    y = fused.forward(xt)
    assert torch.equal(y, multi.forward(xt))
    assert fused.stats() == multi.stats()
    assert np.array_equal(y[0].cpu().numpy(), oplan(n, False, K, L).execute(x[0]))


def test_small_fused_degenerate(oz, monkeypatch):
    n, B = 1024, 4
    x = workloads.draw("uniform", 50, B, n)
    x[1] = 0.0                      # all-zero transform: no slices, no groups
    x[2] = x[2].real                # imaginary part zero: part 1 has no slices
    x[3, 17] = complex(np.inf, 0)   # non-finite: NaN output, flagged
    xt = torch.from_numpy(x).cuda()
    fused, multi = plans(oz, monkeypatch, n, B)
    y = fused.forward(xt)
    ym = multi.forward(xt)
    yn = y.cpu().numpy()
    assert np.array_equal(yn[:3], ym[:3].cpu().numpy())
    assert np.all(np.isnan(yn[3])) and np.all(np.isnan(ym[3].cpu().numpy()))
    assert np.all(yn[1] == 0)
    st = fused.stats()
    assert st == multi.stats() and st["nonfinite"] == 1
    op = oplan(n)
    for b in range(3):
        assert np.array_equal(yn[b], op.execute(x[b])), b


def test_small_fused_graph_replay(oz):
    # the c1 configuration through the captured-graph path (second execute onward)
    x = workloads.draw("uniform", 0, 1, 1024)
    xt = torch.from_numpy(x).cuda()
    plan = oz.Plan(1024, 1)
    out = torch.empty_like(xt)
    ref = oplan(1024).execute(x[0])
    for _ in range(4):
        plan.forward(xt, out=out)
        assert np.array_equal(out[0].cpu().numpy(), ref)
