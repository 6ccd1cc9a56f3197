"""Multi-GPU helpers (one process per GPU, torch.distributed over NCCL / NVLink).

Two partitionings of the hot path:

* Batch sharding -- transforms are independent units, so rank r simply owns a
  contiguous slice of the batch; no collective touches the data path.
* One large transform -- the 8 units (prime q, real convolution cv) of Alg.8
  (u = 2 cv + q) are split into contiguous blocks of 8 / world units.  Every rank
  redoes the O(n) premultiply + split (identical digits everywhere), computes the
  forward NTTs, NTT-domain accumulation and inverse NTTs of its units, and the
  residues [8 units][g groups][n] (g = the schedule's largest group count, known to every
  rank after the split) are all-gathered in place (one NCCL all_gather_into_tensor)
  before every rank runs Garner's CRT, the DD recombination and the post-chirp.

The compute steps are passed in as callables so the gather/layout logic can be tested
with the CPU oracle under the gloo backend (tests/test_dist_gloo.py); on GPUs they are
Plan.shard_partial / Plan.shard_finish.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

NUNITS = 8  # 2 primes x 4 real convolutions


def batch_slice(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, start + count) of `total` independent transforms for `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def shard_units(rank: int, world: int) -> list[int]:
    """Units u = 2*cv + q owned by `rank` (contiguous block; world must divide 8)."""
    if NUNITS % world:
        raise ValueError("world size must divide 8 for single-transform sharding")
    per = NUNITS // world
    return list(range(rank * per, (rank + 1) * per))


def unit_of(cv: int, q: int) -> int:
    return 2 * cv + q


def sharded_transform(residues: torch.Tensor, n: int, rank: int, world: int,
                      partial: Callable[[int, int, torch.Tensor], int],
                      finish: Callable[[torch.Tensor, int], torch.Tensor],
                      group=None) -> torch.Tensor:
    """Run one length-n transform split over `world` ranks.

    residues: flat buffer of at least 8 * K*K * n words on this rank's device.
    partial(rank, world, residues) writes this rank's units into their place of the layout
    [8 units][g][n] and returns g (the schedule's group count, the same on every rank);
    one in-place all_gather_into_tensor of the equal rank slices completes the 8 g n words
    on every rank (no staging copy); finish(residues, g) returns the transform.
    """
    g = partial(rank, world, residues)
    if world > 1:
        buf = residues[:NUNITS * g * n]
        per = buf.numel() // world
        dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per], group=group)
    return finish(residues, g)


def gpu_sharded_forward(plan, x: torch.Tensor, rank: int, world: int, direction: int = -1,
                        group=None) -> torch.Tensor:
    """Single-transform sharded execute on GPUs (transform 0 of x)."""
    residues = torch.empty(plan.shard_residue_bytes() // 4, dtype=torch.int32, device=x.device)
    out = torch.empty(plan.n, dtype=torch.complex128, device=x.device)

    def partial(r, w, res):
        return plan.shard_partial(x, r, w, res, direction)

    def finish(res, g):
        return plan.shard_finish(res, g, out, direction)

    return sharded_transform(residues, plan.n, rank, world, partial, finish, group)
