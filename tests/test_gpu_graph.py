"""ozfft_execute's CUDA-graph path (plans with batch * m <= 2^25): the first execute with a
given (in, out, direction) launches directly, the second captures a graph, later ones
replay it.  Every call must give the same bits and count the same kernel launches; buffers
that change every call never get a graph but still compute correctly."""
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    oz.load_library()
    return oz


@pytest.mark.parametrize("n,B", [(1000, 1), (3001, 4), (1 << 14, 8)])
def test_graph_capture_replay(oz, n, B):
    x = torch.from_numpy(workloads.draw("normal", n, B, n)).cuda()
    plan = oz.Plan(n, B)
    out = torch.empty_like(x)
    ref = None
    counts = []
    for _ in range(4):  # direct, capture, replay, replay
        l0 = oz.kernel_launches()
        plan.forward(x, out=out)
        torch.cuda.synchronize()
        counts.append(oz.kernel_launches() - l0)
        if ref is None:
            ref = out.clone()
        assert torch.equal(out, ref)
    assert len(set(counts)) == 1 and counts[0] > 0, counts
    # new input values in the same buffer: the replayed graph reads them
    x2 = torch.from_numpy(workloads.draw("uniform", n + 1, B, n)).cuda()
    x.copy_(x2)
    plan.forward(x, out=out)
    fresh = oz.Plan(n, B).forward(x2)
    assert torch.equal(out, fresh)
    # the inverse direction is its own key
    inv_ref = oz.Plan(n, B).inverse(fresh)
    buf = torch.empty_like(x)
    for _ in range(3):
        plan.inverse(out, out=buf)
        assert torch.equal(buf, inv_ref)


def test_changing_buffers(oz):
    n, B = 2000, 2
    plan = oz.Plan(n, B)
    xs = [torch.from_numpy(workloads.draw("signexp", 50 + i, B, n)).cuda() for i in range(12)]
    refs = [oz.Plan(n, B).forward(x) for x in xs]
    for _ in range(2):
        for x, r in zip(xs, refs):
            assert torch.equal(plan.forward(x), r)  # new output buffer every call


def test_rebind_drops_graphs(oz):
    """Re-binding the plan to new persistent / workspace buffers (ozfft_plan_bind again)
    must not replay graphs captured against the old ones."""
    n, B = 3000, 2
    x = torch.from_numpy(workloads.draw("normal", 91, B, n)).cuda()
    plan = oz.Plan(n, B)
    out = torch.empty_like(x)
    for _ in range(3):  # direct, capture, replay
        plan.forward(x, out=out)
    ref = out.clone()
    old_ws, old_pers = plan.workspace, plan.persistent
    plan.persistent = torch.empty_like(plan.persistent)
    plan.workspace = torch.empty_like(plan.workspace)
    lib = oz.load_library()
    rc = lib.ozfft_plan_bind(plan._h, plan.persistent.data_ptr(), plan.persistent.numel(),
                             plan.workspace.data_ptr(), plan.workspace.numel(), None)
    assert rc == 0
    old_ws.fill_(0xFF)
    old_pers.fill_(0xFF)  # a stale graph would read garbage tables (twiddles, W, chirp)
    for _ in range(3):
        out.zero_()
        plan.forward(x, out=out)
        assert torch.equal(out, ref)
