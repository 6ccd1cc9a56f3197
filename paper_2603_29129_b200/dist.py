"""Multi-GPU helpers (one process per GPU, torch.distributed over NCCL / NVLink).

Two partitionings of the hot path:

* Batch sharding -- transforms are independent units, so rank r simply owns a
  contiguous slice of the batch; no collective touches the data path.
* One large transform -- the 8 units (prime q, real convolution cv) of Alg.8
  (u = 2 cv + q) are split into contiguous blocks of 8 / world units.  Every rank
  redoes the O(n) premultiply + split (identical digits everywhere), computes the
  forward NTTs, NTT-domain accumulation and inverse NTTs of its units, and the
  residues [8 units][K*K groups][n] are all-gathered (one NCCL all_gather_into_tensor)
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


def sharded_transform(residues: torch.Tensor, rank: int, world: int,
                      partial: Callable[[int, int, torch.Tensor], None],
                      finish: Callable[[torch.Tensor], torch.Tensor],
                      group=None) -> torch.Tensor:
    """Run one transform split over `world` ranks.

    residues: flat int32 buffer of 8 * G * n words (layout [unit][group][n]) on this
    rank's device; partial(rank, world, residues) fills this rank's contiguous slice;
    finish(residues) returns the transform from the gathered buffer.
    """
    partial(rank, world, residues)
    if world > 1:
        per = residues.numel() // world
        mine = residues[rank * per:(rank + 1) * per].clone()
        dist.all_gather_into_tensor(residues, mine, group=group)
    return finish(residues)


def gpu_sharded_forward(plan, x: torch.Tensor, rank: int, world: int, direction: int = -1,
                        group=None) -> torch.Tensor:
    """Single-transform sharded execute on GPUs (plan.batch transforms; transform 0 used)."""
    nwords = plan.shard_residue_bytes() // 4
    residues = torch.empty(nwords, dtype=torch.int32, device=x.device)
    out = torch.empty(plan.n, dtype=torch.complex128, device=x.device)

    def partial(r, w, res):
        plan.shard_partial(x, r, w, res, direction)

    def finish(res):
        return plan.shard_finish(res, out, direction)

    return sharded_transform(residues, rank, world, partial, finish, group)
