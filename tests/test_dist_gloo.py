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
        # exchange sized by the schedule: g = max_cv ng_cv (every rank knows it after the
        # split), layout [8 units][g][n] inside a K*K-capacity buffer
        g = int(max(taps["sched"][cv, 0] for cv in range(4)))
        assert 5 <= g <= G  # >= 2K - 1 anti-diagonal groups; Alg.8 gaps add groups (n = 37: 7)
        buf = torch.full((D.NUNITS * G * n,), -1, dtype=torch.int64)

        def partial(r, w, res):
            for u in D.shard_units(r, w):
                res[:D.NUNITS * g * n].view(D.NUNITS, g, n)[u] = torch.from_numpy(full[u][:g])
            return g

        def finish(res, gg):
            return res[:D.NUNITS * gg * n].view(D.NUNITS, gg, n).clone()

        got = D.sharded_transform(buf, n, rank, world, partial, finish)
        assert np.array_equal(got.numpy(), full[:, :g])
        assert torch.all(buf[D.NUNITS * g * n:] == -1)  # nothing beyond the 8 g n words moved
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


def test_bench_rank_inputs_cover_the_config():
    """bench.py's batch sharding: the ranks' row slices of the seeded config input concatenate
    to exactly workloads.config_input(cfg) (every rank transforms part of the N = 1 job)."""
    import bench
    for name in ("c1", "c2", "c3", "c4"):
        cfg = workloads.CONFIGS[name]
        full = workloads.config_input(cfg)
        for world in (1, 2, 3, 4, 8):
            parts = [bench.rank_input(cfg, r, world) for r in range(world)]
            assert [p[0] for p in parts] == [D.batch_slice(cfg.batch, r, world)[0] for r in range(world)]
            cat = np.concatenate([p[2] for p in parts if p[1]])
            assert cat.shape == full.shape and np.array_equal(cat, full), (name, world)


def _gather_worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        total, n = 7, 5
        full = torch.from_numpy(workloads.draw("normal", 3, total, n))
        start, cnt = D.batch_slice(total, rank, world)
        coll = bench.Coll(world, torch.device("cpu"))
        got = coll.gather_rows(full[start:start + cnt].clone() if cnt else None, total, n)
        assert torch.equal(got, full)
        assert coll.max(float(rank)) == float(world - 1)
        outq.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        outq.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_gather_rows_gloo(world):
    """bench.Coll.gather_rows reassembles the ranks' output rows in batch order (the
    bitwise_vs_n1 check), including ranks with unequal counts."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res
