"""Multi-GPU sharding of the all-pairs passes.

Both all-pairs passes enumerate an upper-triangular space of tile-pair units
(``glr_*_units``).  Rank g of G takes the contiguous range
[floor(gU/G), floor((g+1)U/G)); units have equal cost (diagonal ones half), so
the static split is balanced to within one unit.  Inputs are replicated (each
rank holds xy/edges: 24 + 64 MB for C5), every rank computes its partial
(count, dev_sum, occlusion count) on its own device with no data-path
collective, and ONE allreduce(sum) of a float64[3] buffer combines them --
counts stay exact below 2^53.

The reference has no distributed path; its only parallel
invariant is that results do not depend on the worker count
(engine.py:243-247), which ``tests/test_sharding.py`` checks for 1 and 2
ranks.
"""

from __future__ import annotations

from dataclasses import dataclass


def shard_range(units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous unit range of ``rank`` among ``world`` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return units * rank // world, units * (rank + 1) // world


def shard_plan(units: int, world: int) -> list[tuple[int, int]]:
    plan = [shard_range(units, r, world) for r in range(world)]
    # cross-check (per-GPU unit ranges must tile [0, U))
    assert plan[0][0] == 0 and plan[-1][1] == units
    assert all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
    return plan


@dataclass
class Partial:
    """One rank's contribution; fields add across ranks."""

    crossings: float = 0.0
    dev_sum: float = 0.0
    occlusions: float = 0.0

    def as_list(self) -> list[float]:
        return [self.crossings, self.dev_sum, self.occlusions]


def allreduce_partials(buf, group=None):
    """Sum a float64[3] (count, dev, occlusions) tensor over the process
    group in place (NCCL on GPU ranks, gloo in the CPU tests)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def sharded_evaluate(dg, radius: float | None, ideal: float | None, rank: int, world: int,
                     with_crossing: bool = True, records=None, out=None,
                     strategy: str = "dense"):
    """Compute this rank's partial (count, dev_sum, occlusions) on the current
    CUDA device into a device float64[3] tensor and allreduce it.  Returns the
    tensor (summed over ranks); no host synchronisation.  ``strategy`` as in
    metrics (dense unit triangle or culled candidate list); every rank builds
    the same plan, so the unit spaces agree."""
    import torch

    from . import metrics as M

    if out is None:
        out = torch.zeros(3, dtype=torch.float64, device=dg.xy.device)
    else:
        out.zero_()
    if with_crossing and dg.num_edges >= 2:
        rec = records if records is not None else M.CrossingRecords(dg, strategy)
        b, e = shard_range(rec.units, rank, world)
        rec.partial(ideal, b, e, out=out[0:2])
    if radius is not None and dg.num_vertices >= 2:
        plan = M.OcclusionPlan(dg, radius, strategy)
        b, e = shard_range(plan.units, rank, world)
        plan.partial(b, e, out=out[2:3])
    return allreduce_partials(out)
