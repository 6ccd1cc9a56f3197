"""Single-transform sharding on one GPU: the ranks' shard_partial calls are
run one after the other (no rank waits on another), their unit slices fill the residue
buffer, shard_finish reconstructs -- bit-identical to the unsharded execute and the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1000, 5000, 1 << 14])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_roundtrip(n, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    x = torch.from_numpy(workloads.draw("uniform", n + world, 1, n)).cuda()
    plan = oz.Plan(n, 1)
    ref = plan.forward(x)[0]
    res = torch.zeros(plan.shard_residue_bytes() // 4, dtype=torch.int32, device="cuda")
    assert plan.shard_residue_bytes() == 8 * 9 * n * 4  # K*K capacity
    gs = {plan.shard_partial(x, r, world, res) for r in range(world)}
    assert len(gs) == 1
    g = gs.pop()
    if world > 1:  # exchange sized by the schedule: 2K - 1 groups per conv for these inputs
        assert g == 5 and plan.shard_residue_bytes(g) == 160 * n
    out = torch.empty(n, dtype=torch.complex128, device="cuda")
    plan.shard_finish(res, g, out)
    assert torch.equal(out, ref)
    assert np.array_equal(out.cpu().numpy(), O.Plan(n).execute(x[0].cpu().numpy()))
    # inverse direction through the same path
    yi = plan.inverse(x)[0]
    for r in range(world):
        g = plan.shard_partial(x, r, world, res, direction=+1)
    plan.shard_finish(res, g, out, direction=+1)
    assert torch.equal(out, yi)


def test_shard_schedule_with_gaps():
    """phi = 4 inputs (Alg.8 gaps in the TS-like regime are rare in DD, but K = 4, L = 2
    splits the anti-diagonals): the exchange stride follows the largest group count."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    n = 3000
    x = torch.from_numpy(workloads.phi_input(n, 4.0, seed=77, batch=1)).cuda()
    plan = oz.Plan(n, 1, K=4, L=2)
    ref = plan.forward(x)[0]
    res = torch.zeros(plan.shard_residue_bytes() // 4, dtype=torch.int32, device="cuda")
    for world in (2, 8):
        gs = {plan.shard_partial(x, r, world, res) for r in range(world)}
        assert len(gs) == 1
        g = gs.pop()
        st = plan.stats()
        assert 1 <= g <= 16
        out = torch.empty(n, dtype=torch.complex128, device="cuda")
        plan.shard_finish(res, g, out)
        assert torch.equal(out, ref)


@pytest.mark.parametrize("world", [1, 8])
def test_shard_c3_size_and_nonfinite(world):
    """The single-transform variant at the c3 length (n = 2^18: the finish from gathered
    residues runs k_crt_dd + k_finish_dd) equals the batched execute bit for bit; a
    non-finite input gives NaN through the same path."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    n = 1 << 18
    x = torch.from_numpy(workloads.draw("uniform", 2, 1, n)).cuda()
    plan = oz.Plan(n, 1)
    ref = plan.forward(x)[0]
    res = torch.zeros(plan.shard_residue_bytes() // 4, dtype=torch.int32, device="cuda")
    out = torch.empty(n, dtype=torch.complex128, device="cuda")
    for r in range(world):
        g = plan.shard_partial(x, r, world, res)
    plan.shard_finish(res, g, out)
    assert torch.equal(out, ref)
    x[0, 12345] = float("nan")
    for r in range(world):
        g = plan.shard_partial(x, r, world, res)
    plan.shard_finish(res, g, out)
    assert torch.isnan(out.real).all() and torch.isnan(out.imag).all()
