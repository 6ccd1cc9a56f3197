"""Fault injection: a single flipped bit in one NTT-domain group value
(OZFFT_FAULT_INJECT=1, read at plan create) must trip the bit-exact comparison against the
oracle -- the parity tests can fail, so their passing means something."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1000, 5000])  # one-pass (residues) and two-pass (G) plans
def test_fault_is_caught(monkeypatch, n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    from test_gpu_parity import check_taps
    x = workloads.draw("uniform", 3, 1, n)
    xt = torch.from_numpy(x).cuda()
    yo, ot = O.Plan(n).execute(x[0], taps=True)
    clean = oz.Plan(n, 1)
    y0, t0 = clean.execute_taps(xt)
    check_taps(t0, ot, n, 3, 0)  # the clean plan matches
    assert np.array_equal(y0[0].cpu().numpy(), yo)
    monkeypatch.setenv("OZFFT_FAULT_INJECT", "1")
    bad = oz.Plan(n, 1)
    y1, t1 = bad.execute_taps(xt)
    with pytest.raises(AssertionError):
        check_taps(t1, ot, n, 3, 0)
    assert not np.array_equal(y1[0].cpu().numpy(), yo)
    ng = int(ot["sched"][0, 0])
    assert not np.array_equal(t1["crt"][0, 0, ng - 1].cpu().numpy(), ot["crt"][0, ng - 1])
    # the device-buffer execute path too
    assert not torch.equal(bad.forward(xt), clean.forward(xt))
