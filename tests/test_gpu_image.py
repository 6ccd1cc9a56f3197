"""GPU parity of the complex-image accumulation plans (accum="image")
against the oracle's image mode (oracle.Plan(..., image=True)), through the C ABI.

Bar: digits, shared exponents, image spectra X and W, accumulated image groups Z,
inverse-NTT residues of both images, Re / Im CRT integers and the complex schedule
bit-exact; fp64 output bitwise equal.  Sizes: one-pass rows, two-pass plans, pruned and
unpruned (cyclic) last column stage, ragged / prime n, and BASELINE configs sampled as in
tests/test_gpu_configs.py.
"""
import functools

import numpy as np
import pytest
import torch

import oracle as O
import workloads
from test_gpu_configs import sample

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    oz.load_library()
    return oz


@functools.lru_cache(maxsize=8)
def oplan(n, cyclic=False, K=3, L=3):
    return O.Plan(n, K, L, image=True, cyclic=cyclic)


def check_image_taps(gt, ot, b):
    g = {k: v[b].cpu().numpy() for k, v in gt.items() if k != "W"}
    assert np.array_equal(g["kv"], ot["kv"]) and g["kv"][0] == g["kv"][1]
    k = int(ot["kv"][0])
    assert np.array_equal(g["E"][:, :k], ot["E"][:, :k])
    assert np.array_equal(g["digits"][:, :k], ot["digits"][:, :k])
    assert np.array_equal(g["X"][:, :k].astype(np.uint32), ot["X"][:, :k])
    assert np.array_equal(g["sched"], ot["sched"])
    ng = int(ot["sched"][0, 0])
    for img in range(2):
        assert np.array_equal(g["Z"][img, :ng].astype(np.uint32), ot["Z"][img, :ng]), img
        assert np.array_equal(g["res"][img, :ng].astype(np.uint32), ot["res"][img, :ng]), img
    for part in range(2):
        assert np.array_equal(g["crt"][part, :ng], ot["crt"][part, :ng]), part


@pytest.mark.parametrize("n,B,dist,seed,cyclic", [
    (1, 1, "uniform", 0, False), (2, 2, "normal", 1, False), (5, 3, "signexp", 2, False),
    (100, 2, "uniform", 3, False), (1024, 1, "normal", 4, False), (2047, 2, "signexp", 5, False),
    (3001, 2, "normal", 6, False), (1 << 13, 1, "uniform", 7, False),
    (1 << 13, 2, "signexp", 8, True), (1 << 15, 1, "normal", 9, True)])
def test_image_taps_bit_exact(oz, n, B, dist, seed, cyclic):
    x = workloads.draw(dist, seed, B, n)
    plan = oz.Plan(n, B, accum="image", conv="cyclic" if cyclic else "padded")
    op = oplan(n, cyclic)
    assert plan.m == op.m and plan.alpha == op.alpha
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    assert np.array_equal(gt["W"].cpu().numpy().astype(np.uint32), op.tables()["W"])
    yg = y.cpu().numpy()
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        check_image_taps(gt, ot, b)
        assert np.array_equal(yg[b], yo)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_image_configs(oz, name):
    cfg = workloads.CONFIGS[name]
    x = workloads.config_input(cfg)
    plan = oz.Plan(cfg.n, cfg.batch, accum="image")
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    idx = sample(cfg.batch, seed=2)[:4]
    ys, _ = oplan(cfg.n).execute_batch(np.ascontiguousarray(x[idx]))
    for i, b in enumerate(idx):
        assert np.array_equal(y[b], ys[i]), (name, b)
    st = plan.stats()
    assert st["fwd_ntts"] == 12 * cfg.batch  # 2 images x 3 slices x 2 primes
    if name != "c4":  # uniform / normal inputs: no gaps, 5 groups per image and prime
        assert st["inv_ntts"] == 20 * cfg.batch


def test_image_roundtrip_edges_and_errors(oz):
    n, B = 1000, 4
    x = workloads.draw("normal", 12, B, n)
    x[2, 17] = np.nan
    x[3] = 0.0
    plan = oz.Plan(n, B, accum="image")
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt)
    yn = y.cpu().numpy()
    assert np.all(np.isnan(yn[2])) and np.all(yn[3] == 0)
    op = oplan(n)
    for b in (0, 1):
        assert np.array_equal(yn[b], op.execute(x[b]))
        xr = plan.inverse(y).cpu().numpy()[b]
        assert np.array_equal(xr, op.execute(yn[b], inverse=True))
        assert np.max(np.abs(xr - x[b])) / np.max(np.abs(x[b])) <= 1e-15
    with pytest.raises(oz.OzfftError):
        plan.shard_partial(xt[:1].contiguous(), 0, 2, torch.empty(plan.shard_residue_bytes() // 4,
                                                                   dtype=torch.int32, device="cuda"))


def test_image_error_vs_float128(oz):
    for n, dist in ((1024, "uniform"), (999, "signexp"), (4096, "normal")):
        x = workloads.draw(dist, n, 1, n)
        y = oz.Plan(n, 1, accum="image").forward(torch.from_numpy(x).cuda()).cpu().numpy()[0]
        hi, lo = O.dft_f128(x[0])
        err = np.max(np.abs((y - hi) - lo)) / np.max(np.abs(hi))
        assert err <= 1e-15, (n, err)
