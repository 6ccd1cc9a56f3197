"""Single-transform sharding with the exchange fused into the producing kernels (peer-memory
epilogue, ozfft_shard_partial_p2p, include/ozfft.h): every rank's inverse-NTT
epilogue stores its units' residues into every rank's exchange buffer, and no collective
runs afterwards.  On this one-GPU pool the ranks run on one device: (1) in one process, the
"ranks'" buffers are plain allocations and the partials run one after another -- every
buffer must end complete and finish to the batched execute bit for bit; (2) two processes
on cuda:0 exchange CUDA IPC handles over a gloo group, write into each other's buffers,
meet at a host barrier (no kernel waits on another rank) and finish independently."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1000, 5000, 1 << 18])   # one-pass (row-kernel epilogue), two-pass
@pytest.mark.parametrize("world", [2, 8])
def test_p2p_in_process(n, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_29129_b200 as oz
    x = torch.from_numpy(workloads.draw("normal", 7 * n + world, 1, n)).cuda()
    plan = oz.Plan(n, 1)
    ref = plan.forward(x)[0]
    bufs = [torch.full((plan.shard_residue_bytes() // 4,), -1, dtype=torch.int32, device="cuda")
            for _ in range(world)]
    gs = {plan.shard_partial_p2p(x, r, world, bufs) for r in range(world)}
    assert len(gs) == 1
    g = gs.pop()
    out = torch.empty(n, dtype=torch.complex128, device="cuda")
    used = 8 * g * n
    for r in range(world):  # every rank's buffer was completed by the other ranks' kernels
        assert torch.equal(bufs[r][:used], bufs[0][:used])
        plan.shard_finish(bufs[r], g, out)
        assert torch.equal(out, ref), r
    if n <= 5000:
        assert np.array_equal(out.cpu().numpy(), O.Plan(n).execute(x[0].cpu().numpy()))
    # the NCCL-style path (each rank writes only its own slice) gives the same buffer
    res = torch.zeros_like(bufs[0])
    for r in range(world):
        plan.shard_partial(x, r, world, res)
    assert torch.equal(res[:used], bufs[0][:used])


def _ipc_worker(rank, world, port, n, q):
    import torch.distributed as dist
    import paper_2603_29129_b200 as oz
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        x = torch.from_numpy(workloads.draw("uniform", 11, 1, n)).cuda()
        plan = oz.Plan(n, 1)
        mine = torch.zeros(plan.shard_residue_bytes() // 4, dtype=torch.int32, device="cuda")
        handles = [None] * world
        dist.all_gather_object(handles, oz.ipc_handle(mine))
        ptrs = [mine.data_ptr() if r == rank else oz.ipc_open(handles[r]) for r in range(world)]
        for direction in (-1, +1):
            g = plan.shard_partial_p2p(x, rank, world, ptrs, direction=direction)
            torch.cuda.synchronize()
            dist.barrier()  # every rank's kernels (and their stores into `mine`) completed
            out = torch.empty(n, dtype=torch.complex128, device="cuda")
            plan.shard_finish(mine, g, out, direction=direction)
            ref = plan.execute(x, direction)[0]
            q.put((rank, direction, bool(torch.equal(out, ref))))
            dist.barrier()  # nobody rewrites a buffer another rank still reads
        torch.cuda.synchronize()
        dist.barrier()
        for r in range(world):
            if r != rank:
                oz.ipc_close(ptrs[r], handles[r])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 5000])
def test_p2p_two_processes_ipc(n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    got = sorted(q.get(timeout=10) for _ in range(4))
    assert got == [(0, -1, True), (0, 1, True), (1, -1, True), (1, 1, True)], got
