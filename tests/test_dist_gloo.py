"""Multi-process (world_size 2 and 4, gloo on 127.0.0.1) tests of the host-side sharding
logic of paper_2603_29129_b200.dist, driven by the CPU oracle (no GPU):

* batch sharding covers the global batch exactly once and each rank's transforms
  match the oracle run on the full batch;
* single-transform sharding: each rank fills its unit slice of the residue buffer
  [8 units][K*K][n] from the oracle's inverse-NTT taps, one all_gather_into_tensor
  assembles the buffer, and the result equals the oracle's residues for every unit;
* the max-over-ranks reduction used by bench.py for timing.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads
from paper_2603_29129_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, K, L = 37, 3, 3
        G = K * K
        plan = O.Plan(n, K, L)
        # ---- batch sharding
        total = 7
        x_all = workloads.draw("normal", 5, total, n)
        start, cnt = D.batch_slice(total, rank, world)
        mine = [plan.execute(x_all[b]) for b in range(start, start + cnt)]
        counts = torch.tensor([cnt], dtype=torch.int64)
        dist.all_reduce(counts)
        assert counts.item() == total
        ref = [plan.execute(x_all[b]) for b in range(total)]
        for i, b in enumerate(range(start, start + cnt)):
            assert np.array_equal(mine[i], ref[b])
        # ---- single transform: units (cv, q) sharded, residues all-gathered
        x = workloads.draw("uniform", 9, 1, n)[0]
        _, taps = plan.execute(x, taps=True)
        full = np.zeros((D.NUNITS, G, n), np.int64)
        for cv in range(4):
            for qq in range(2):
                full[D.unit_of(cv, qq)] = taps["res"][cv, :, qq, :]
        buf = torch.zeros(D.NUNITS * G * n, dtype=torch.int64)

        def partial(r, w, res):
            for u in D.shard_units(r, w):
                res.view(D.NUNITS, G, n)[u] = torch.from_numpy(full[u])

        def finish(res):
            return res.view(D.NUNITS, G, n).clone()

        got = D.sharded_transform(buf, rank, world, partial, finish)
        assert np.array_equal(got.numpy(), full)
        # ---- max over ranks (bench.py timing rule)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == float(world)
        outq.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        outq.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res


def test_partition_helpers():
    for total in (1, 7, 16, 1024):
        for world in (1, 2, 3, 8):
            spans = [D.batch_slice(total, r, world) for r in range(world)]
            covered = [i for s, c in spans for i in range(s, s + c)]
            assert covered == list(range(total))
    assert D.shard_units(3, 8) == [3]
    assert D.shard_units(1, 2) == [4, 5, 6, 7]
    with pytest.raises(ValueError):
        D.shard_units(0, 3)
