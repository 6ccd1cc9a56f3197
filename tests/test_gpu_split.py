"""The one-launch split (k_split_cluster, n <= 2^15: a1 + a2 with one thread-block cluster per
transform) against the multi-launch split (k_split_max per level +
k_split_digits) and against the oracle.

Bar: digits, exponents, slice counts, schedules and the fp64 output bitwise equal between
the two GPU paths (same per-element operation sequence, exact max), and bitwise equal to
the oracle at the largest cluster length.  OZFFT_SPLIT_CLUSTER_MAXLEN=0 (read at plan
creation) selects the multi-launch path.
"""
import numpy as np
import pytest
import torch

import oracle as O
import workloads
from test_gpu_parity import check_taps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    oz.load_library()
    return oz


def plans(oz, monkeypatch, n, B, **kw):
    fused = oz.Plan(n, B, **kw)
    monkeypatch.setenv("OZFFT_SPLIT_CLUSTER_MAXLEN", "0")
    multi = oz.Plan(n, B, **kw)
    monkeypatch.delenv("OZFFT_SPLIT_CLUSTER_MAXLEN")
    return fused, multi


def same_split(ta, tb):
    for k in ("digits", "E", "kv", "sched", "X", "crt"):
        assert torch.equal(ta[k], tb[k]), k


# ragged cluster chunks (n not a multiple of the cluster size), one- and two-pass plans,
# the 8-CTA cluster cap, and the largest cluster length
@pytest.mark.parametrize("n,B,dist", [
    (1, 2, "uniform"), (7, 3, "normal"), (256, 1, "signexp"), (257, 2, "uniform"),
    (1000, 2, "normal"), (2049, 2, "signexp"), (4097, 1, "uniform"), (16384, 2, "normal"),
    (30011, 1, "signexp"), (32768, 1, "normal")])
@pytest.mark.parametrize("mode", [{}, {"precision": "ts"}, {"accum": "image"}, {"conv": "cyclic"}])
def test_cluster_split_matches_multi_launch(oz, monkeypatch, n, B, dist, mode):
    if mode.get("conv") == "cyclic" and (n & (n - 1) or n < 4):
        pytest.skip("cyclic plans need a power-of-two n")
    x = torch.from_numpy(workloads.draw(dist, n + 3, B, n)).cuda()
    fused, multi = plans(oz, monkeypatch, n, B, **mode)
    ya, ta = fused.execute_taps(x)
    yb, tb = multi.execute_taps(x)
    same_split(ta, tb)
    assert torch.equal(ya, yb)
    # and the production (non-tap) path, forward and inverse
    assert torch.equal(fused.forward(x), multi.forward(x))
    assert torch.equal(fused.inverse(x), multi.inverse(x))


def test_cluster_split_nonfinite(oz, monkeypatch):
    """A non-finite transform in a batch: both paths flag it (kv = 0, NaN output) and leave
    the finite transforms bitwise equal."""
    n, B = 3000, 3
    x = workloads.draw("normal", 5, B, n)
    x[1, 17] = np.inf + 0j
    xd = torch.from_numpy(x).cuda()
    fused, multi = plans(oz, monkeypatch, n, B)
    ya, ta = fused.execute_taps(xd)
    yb, tb = multi.execute_taps(xd)
    assert torch.equal(ta["kv"], tb["kv"]) and ta["kv"][1].sum() == 0
    assert torch.equal(ta["sched"], tb["sched"]) and torch.equal(ta["E"], tb["E"])
    for b in (0, 2):
        assert torch.equal(ya[b], yb[b])
        assert torch.equal(ta["digits"][b], tb["digits"][b])
    assert torch.isnan(ya[1]).all() and torch.isnan(yb[1]).all()
    assert fused.stats()["nonfinite"] == multi.stats()["nonfinite"] == 1


def test_cluster_split_largest_vs_oracle(oz):
    """n = 2^15 (8 CTAs of 4096 elements): taps bit-exact against the oracle."""
    n = 1 << 15
    x = workloads.draw("uniform", 77, 1, n)
    plan = oz.Plan(n, 1)
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    yo, ot = O.Plan(n).execute(x[0], taps=True)
    check_taps(gt, ot, n, 3, 0)
    assert np.array_equal(y[0].cpu().numpy(), yo)
