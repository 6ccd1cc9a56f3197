"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): integer stages bit-exact (digits, exponents, slice
counts, forward spectra X, cached W spectra, accumulated groups Z, inverse-NTT
residues, CRT integers, Alg.8 schedules); fp64 output within 1e-15 max
relative-to-norm of the oracle (both sides run the same DD op sequence, so the
output is expected to be bitwise equal -- asserted separately where it holds).
"""
import functools

import numpy as np
import pytest
import torch

import oracle as O
import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-15  # north_star: max relative-to-norm error vs the oracle


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    oz.load_library()
    return oz


@functools.lru_cache(maxsize=16)
def oplan(n, K=3, L=3):
    return O.Plan(n, K, L)


def rel_norm_err(a, b):
    d = np.max(np.abs(a - b))
    s = np.max(np.abs(b))
    return d / s if s > 0 else d


def check_taps(gt, ot, n, L, b_idx=0):
    """Compare one transform's GPU taps (gt, batch index b_idx) with oracle taps ot."""
    g = {k: v[b_idx].cpu().numpy() if k != "W" else v.cpu().numpy() for k, v in gt.items()}
    assert np.array_equal(g["kv"], ot["kv"])
    kv = ot["kv"]
    for a in range(2):
        assert np.array_equal(g["E"][a, :kv[a]], ot["E"][a, :kv[a]])
        assert np.array_equal(g["digits"][a, :kv[a]], ot["digits"][a, :kv[a]])
        assert np.array_equal(g["X"][a, :kv[a]].astype(np.uint32), ot["X"][a, :kv[a]])
    assert np.array_equal(g["sched"], ot["sched"])
    for cv in range(4):
        ng = int(ot["sched"][cv, 0])
        assert np.array_equal(g["Z"][cv, :ng].astype(np.uint32), ot["Z"][cv, :ng]), cv
        assert np.array_equal(g["res"][cv, :ng].astype(np.uint32), ot["res"][cv, :ng]), cv
        assert np.array_equal(g["crt"][cv, :ng], ot["crt"][cv, :ng]), cv


# sizes: single pass (m <= 4096), two passes (m >= 8192), ragged / prime n, tiny n
@pytest.mark.parametrize("n,B,dist,seed", [
    (1, 1, "uniform", 0), (2, 2, "normal", 1), (3, 1, "signexp", 2), (5, 3, "uniform", 3),
    (16, 2, "normal", 4), (37, 1, "signexp", 5), (100, 2, "uniform", 6), (1000, 2, "normal", 7),
    (1024, 1, "uniform", 0), (2047, 1, "signexp", 8), (3001, 2, "normal", 9),
    (5000, 1, "uniform", 10), (1 << 13, 2, "signexp", 11)])
def test_taps_bit_exact(oz, n, B, dist, seed):
    x = workloads.draw(dist, seed, B, n)
    plan = oz.Plan(n, B)
    op = oplan(n)
    assert plan.m == op.m and plan.alpha == op.alpha
    xt = torch.from_numpy(x).cuda()
    y, gt = plan.execute_taps(xt)
    tab = op.tables()
    assert np.array_equal(gt["W"].cpu().numpy().astype(np.uint32), tab["W"])
    st = plan.stats()
    assert st["k"][2:] == list(tab["kw"])
    yg = y.cpu().numpy()
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        check_taps(gt, ot, n, 3, b)
        assert rel_norm_err(yg[b], yo) <= TOL
        assert np.array_equal(yg[b], yo), "fp64 output not bitwise equal to the oracle"


@pytest.mark.parametrize("K,L", [(1, 1), (2, 1), (3, 1), (3, 2), (4, 3), (8, 8)])
def test_other_K_L(oz, K, L):
    n, B = 700, 2
    x = workloads.phi_input(n, 4.0, seed=K * 10 + L, batch=B)  # wide exponent range
    plan = oz.Plan(n, B, K=K, L=L)
    op = oplan(n, K, L)
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        check_taps(gt, ot, n, L, b)
        assert np.array_equal(y[b].cpu().numpy(), yo)


@pytest.mark.parametrize("n,K,L", [(5000, 8, 8), (5000, 1, 1), (40000, 4, 3), (40000, 8, 2)])
def test_other_K_L_two_pass(oz, n, K, L):
    """Other split caps through the two-pass NTT (column + row kernels; K = 8 is the cap,
    kMaxK) and both split paths (cluster for n <= 2^15, multi-launch above)."""
    x = workloads.phi_input(n, 4.0, seed=n + K * 10 + L, batch=1)
    plan = oz.Plan(n, 1, K=K, L=L)
    assert plan.m >= 8192
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    yo, ot = oplan(n, K, L).execute(x[0], taps=True)
    check_taps(gt, ot, n, L, 0)
    assert np.array_equal(y[0].cpu().numpy(), yo)


def test_edge_cases(oz):
    n = 300
    plan = oz.Plan(n, 4)
    op = oplan(n)
    x = np.zeros((4, n), np.complex128)
    x[1, 0] = 1.0                       # impulse: k_re = 1, k_im = 0 (ruling 11)
    x[2] = workloads.draw("normal", 3, 1, n)[0]
    x[2, 17] = np.nan                   # non-finite -> all-NaN output (ruling 18)
    x[3] = workloads.draw("uniform", 4, 1, n)[0] * 2.0 ** -700  # tiny but in range
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    st = plan.stats()
    assert st["nonfinite"] == 1 and st["flags"] & 1
    assert np.all(y[0] == 0)
    assert np.all(np.isnan(y[2]))
    for b in (1, 3):
        assert np.array_equal(y[b], op.execute(x[b]))
    # in-place (in == out)
    xt = torch.from_numpy(x[[1, 3, 0, 1]].copy()).cuda()
    ref = plan.forward(xt.clone())
    plan.forward(xt, out=xt)
    assert torch.equal(xt, ref)


def test_inverse_and_roundtrip(oz):
    n, B = 1000, 3
    x = workloads.draw("normal", 12, B, n)
    plan = oz.Plan(n, B)
    op = oplan(n)
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt)
    xr = plan.inverse(y).cpu().numpy()
    yn = y.cpu().numpy()
    for b in range(B):
        assert np.array_equal(op.execute(yn[b], inverse=True), xr[b])
        assert rel_norm_err(xr[b], x[b]) <= 1e-15


def test_counts_phi0(oz, golden):
    """52 runtime NTT calls per transform at (K,L)=(3,3), phi=0; 64 with cached."""
    n, B = 4096, 4
    plan = oz.Plan(n, B)
    plan.forward(torch.from_numpy(workloads.phi_input(n, 0.0, 1, B)).cuda())
    st = plan.stats()
    g = golden["ntt_counts"]
    assert st["fwd_ntts"] + st["inv_ntts"] == B * g["K3_L3_runtime"]
    assert st["fwd_ntts"] // B + st["inv_ntts"] // B + st["cached_ntts"] == g["K3_L3_total"]


def test_host_entry_point(oz):
    n, B = 777, 3
    x = workloads.draw("uniform", 5, B, n)
    plan = oz.Plan(n, B)
    xh = torch.from_numpy(x).pin_memory()
    yh = plan.execute_host(xh)
    yd = plan.forward(torch.from_numpy(x).cuda()).cpu()
    assert torch.equal(yh, yd)


@pytest.mark.parametrize("n,B,ws", [(4096, 16, 0), (5000, 13, 20 << 20), (1000, 40, 0), (40000, 16, 0),
                                    (40000, 23, 0)])
def test_host_pipeline_schedules(oz, n, B, ws):
    """execute_host over sub-batches on two compute streams (edge sub-batches, disjoint
    workspace slots, slot reuse when the workspace chunk is smaller than the batch) gives
    the same bits as the device-buffer execute."""
    x = workloads.draw("signexp", B, B, n)
    plan = oz.Plan(n, B, max_workspace_bytes=ws)
    xh = torch.from_numpy(x).pin_memory()
    for _ in range(2):  # the second call reuses the pipeline's streams and events
        yh = plan.execute_host(xh)
    yd = plan.forward(torch.from_numpy(x).cuda()).cpu()
    assert torch.equal(yh, yd)
    xr = plan.execute_host(yh.pin_memory(), direction=+1)
    assert torch.equal(xr, plan.inverse(yd.cuda()).cpu())


def test_chunked_batch(oz):
    """A workspace budget forcing several chunks gives the same bits as one chunk."""
    n, B = 5000, 7
    x = torch.from_numpy(workloads.draw("signexp", 6, B, n)).cuda()
    full = oz.Plan(n, B)
    small = oz.Plan(n, B, max_workspace_bytes=12 << 20)  # chunk 1 (7.2 MB per transform)
    assert small.chunk < B
    assert torch.equal(full.forward(x), small.forward(x))


def test_error_vs_float128(oz):
    """Within 2x the oracle's own error against the __float128 DFT (north_star)."""
    for n, dist in ((1024, "uniform"), (999, "signexp"), (4096, "normal")):
        x = workloads.draw(dist, n, 1, n)
        y = oz.Plan(n, 1).forward(torch.from_numpy(x).cuda()).cpu().numpy()[0]
        yo = oplan(n).execute(x[0])
        hi, lo = O.dft_f128(x[0])
        eo = np.max(np.abs((yo - hi) - lo)) / np.max(np.abs(hi))
        eg = np.max(np.abs((y - hi) - lo)) / np.max(np.abs(hi))
        assert eg <= 2 * eo + 1e-300 and eg <= 1e-15, (n, eg, eo)


@pytest.mark.parametrize("conv,accum,precision", [("padded", "image", "dd"), ("cyclic", "image", "dd"),
                                                  ("padded", "real", "ts"), ("cyclic", "real", "ts")])
def test_modes_chunked_and_host(oz, conv, accum, precision):
    """Every plan mode through the chunked workspace and the host pipeline gives the bits of
    a one-chunk device execute."""
    n, B = 4096, 9
    x = workloads.draw("normal", 31, B, n)
    kw = dict(conv=conv, accum=accum, precision=precision)
    full = oz.Plan(n, B, **kw)
    small = oz.Plan(n, B, max_workspace_bytes=8 << 20, **kw)
    assert small.chunk < B
    xd = torch.from_numpy(x).cuda()
    ref = full.forward(xd)
    assert torch.equal(small.forward(xd), ref)
    assert torch.equal(small.execute_host(torch.from_numpy(x).pin_memory()), ref.cpu())
    assert torch.equal(full.execute_host(torch.from_numpy(x).pin_memory()), ref.cpu())


@pytest.mark.parametrize("p0,p1", [(2013265921, 1811939329), (2130706433, 998244353),
                                   (998244353, 2113929217)])
def test_custom_primes(oz, p0, p1):
    """User-chosen NTT primes (desc.p0 / p1): bit-exact against the oracle with
    the same primes, including p0 > 2 p1 (Garner's z0 mod p1 is a full remainder there)."""
    n, B = 1000, 2
    x = workloads.draw("normal", 17, B, n)
    plan = oz.Plan(n, B, p0=p0, p1=p1)
    op = O.Plan(n, p0=p0, p1=p1)
    assert plan.alpha == op.alpha
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        check_taps(gt, ot, n, 3, b)
        assert np.array_equal(y[b].cpu().numpy(), yo)


@pytest.mark.parametrize("mode", [dict(accum="image"), dict(precision="ts")])
@pytest.mark.parametrize("K,L", [(1, 1), (2, 1), (4, 3), (8, 8)])
def test_modes_other_K_L(oz, mode, K, L):
    """The f2 / f4 plan modes with other split caps and accumulation bounds, wide-range
    inputs (phi = 4): taps and output bit-exact against the oracle's mode."""
    n, B = 700, 2
    x = workloads.phi_input(n, 4.0, seed=K * 10 + L, batch=B)
    plan = oz.Plan(n, B, K=K, L=L, **mode)
    op = O.Plan(n, K, L, image=mode.get("accum") == "image", ts=mode.get("precision") == "ts")
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    for b in range(B):
        yo, ot = op.execute(x[b], taps=True)
        assert np.array_equal(gt["crt"][b].cpu().numpy(), ot["crt"])
        assert np.array_equal(gt["sched"][b].cpu().numpy(), ot["sched"])
        assert np.array_equal(y[b].cpu().numpy(), yo)


def test_huge_batch_tiny_n(oz):
    """batch > 65535 (the gridDim.y limit of the per-transform kernels) runs in chunks."""
    n, B = 5, 70000
    x = workloads.draw("uniform", 5, B, n)
    plan = oz.Plan(n, B)
    assert plan.chunk <= 65535
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    op = O.Plan(n)
    for b in (0, 1, 65534, 65535, 65536, B - 1):
        assert np.array_equal(y[b], op.execute(x[b])), b


@pytest.mark.parametrize("n", [1000, 4096, 1 << 13])
def test_max_digit_input(oz, n):
    """x(j) = conj(omega(j)) makes x' = x (.) omega = |omega|^2 ~ 1 everywhere, so the level-0
    digits of Re x' all sit at the top of the digit range and the group sums approach the
    CRT range bound: bit-exact against the oracle."""
    j = np.arange(n, dtype=np.float64)
    x = np.exp(1j * np.pi * (j * j % (2 * n)) / n)[None, :].astype(np.complex128)
    plan = oz.Plan(n, 1)
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    yo, ot = O.Plan(n).execute(x[0], taps=True)
    d = gt["digits"][0].cpu().numpy()
    # |x'| = 1 up to rounding: mu is 1 or just above, so the level-0 digits are all 2^alpha
    # or all 2^(alpha - 1) (E = 0 or 1)
    assert np.min(np.abs(d[0, 0])) >= 2 ** (plan.alpha - 1) - 1
    check_taps(gt, ot, n, 3, 0)
    assert np.array_equal(y[0].cpu().numpy(), yo)


@pytest.mark.parametrize("seed", range(12))
def test_random_sizes(oz, seed):
    """Seeded random lengths (one- and two-pass, both split paths, prime and composite n)
    and distributions: every tap and the fp64 output bit-exact against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 48000))
    dist = ["uniform", "normal", "signexp"][seed % 3]
    x = workloads.draw(dist, 2000 + seed, 1, n)
    plan = oz.Plan(n, 1)
    y, gt = plan.execute_taps(torch.from_numpy(x).cuda())
    yo, ot = oplan(n).execute(x[0], taps=True)
    check_taps(gt, ot, n, 3, 0)
    assert np.array_equal(y[0].cpu().numpy(), yo), n


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("mode", [dict(precision="ts"), dict(accum="image"), dict(conv="cyclic"),
                                  dict(conv="cyclic", accum="image")])
def test_random_sizes_modes(oz, seed, mode):
    """As test_random_sizes, for the f1 / f2 / f4 plan modes against the oracle's modes."""
    rng = np.random.default_rng(3000 + seed)
    cyc = mode.get("conv") == "cyclic"
    n = 1 << int(rng.integers(2, 16)) if cyc else int(rng.integers(1, 40000))
    x = workloads.draw(["uniform", "normal", "signexp"][seed % 3], 4000 + seed, 1, n)
    plan = oz.Plan(n, 1, **mode)
    op = O.Plan(n, cyclic=cyc, image=mode.get("accum") == "image", ts=mode.get("precision") == "ts")
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y[0], op.execute(x[0])), (n, mode)
