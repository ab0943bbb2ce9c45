"""Multi-GPU sharding of the all-pairs passes.

Both all-pairs passes enumerate an upper-triangular space of tile-pair units
(``glr_*_units``).  Occlusion units have equal cost (diagonal ones half), so
rank g of G takes the contiguous range [floor(gU/G), floor((g+1)U/G)).
Crossing units do not (run reuse makes a j-tile's cost depend on its run
structure), so ``sharded_evaluate`` uses interleaved ownership instead: the
crossing kernel deals units to CTAs in chunks and rank g keeps the chunks
whose index is g (mod G) (``glr_crossing_pairs_interleaved``), which balances
to 1.4% over 8 ranks on C5 with no cost model.  The cost-weighted contiguous
splits further down remain for callers that want contiguous ranges
(``CrossingRecords.shard``).  Inputs are replicated (each
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
    metrics (dense unit triangle or culled candidate list).  Dense: every rank
    holds the same unit triangle and takes interleaved chunks of it.  Culled:
    rank g classifies and scans the tile rows ti = g (mod world) of the
    classified list (``CrossingRecords(rows=...)``); with ``"auto"`` the ranks
    agree on the strategy through one small allreduce of their plan costs."""
    import torch

    from . import metrics as M

    if out is None:
        out = torch.zeros(3, dtype=torch.float64, device=dg.xy.device)
    else:
        out.zero_()
    if with_crossing and dg.num_edges >= 2:
        # culled plans are dealt to the ranks by tile rows, so the plan build
        # (classes, masks) shards with the pass; dense passes by unit chunks
        rec = records if records is not None else M.CrossingRecords(
            dg, strategy, "input" if ideal is None else "theta",
            rows=(rank, world) if world > 1 else None)
        rec.partial_interleaved(ideal, rank, world, out=out[0:2])
    if radius is not None and dg.num_vertices >= 2:
        plan = M.OcclusionPlan(dg, radius, strategy)
        b, e = shard_range(plan.units, rank, world)
        plan.partial(b, e, out=out[2:3])
    return allreduce_partials(out)


# ---- cost-balanced splits ----------------------------------------------------
# Units do not all cost the same: with run reuse (csrc/crossing.cu) a j-tile
# full of run starts costs more than one inside a hub's run.  Measured on C5,
# equal unit counts left the last of 8 ranks 17% slower than the first.  The
# splits below cut the unit sequence at equal cumulative weight instead; every
# rank computes the same cuts from the same weights, so the ranges still tile
# the unit space exactly.

# Extra cost of a run-start j-edge relative to a continuing one.  Calibrated
# on C5 (fused E_c + E_ca, 8 ranges timed back to back on one B200): equal
# unit counts 1.17 max/mean, beta 0.3 -> 1.047, beta 0.6 -> 1.014.
RUN_START_BETA = 0.6


def _cut(cum: "np.ndarray", frac: float) -> int:
    """First index whose cumulative weight reaches frac of the total."""
    import numpy as np

    total = float(cum[-1]) if len(cum) else 0.0
    return int(np.searchsorted(cum, frac * total, side="left"))


def weighted_range(unit_weights, rank: int, world: int) -> tuple[int, int]:
    """Contiguous range of a 1-D unit sequence with per-unit weights."""
    import numpy as np

    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    w = np.asarray(unit_weights, dtype=np.float64)
    U = len(w)
    if U == 0:
        return 0, 0
    cum = np.cumsum(w)
    b = 0 if rank == 0 else min(U, _cut(cum, rank / world) + 1)
    e = U if rank == world - 1 else min(U, _cut(cum, (rank + 1) / world) + 1)
    return b, max(b, e)


def _band_unit_weights(w, band: int):
    """Per-band pieces of the banded unit order (see glr_crossing_band):
    for each band [b0, e): (b0, e, base unit, weight of one full row over the
    band, cumulative weights of the band's triangle rows)."""
    import numpy as np

    T = len(w)
    out = []
    base = 0
    for b0 in range(0, T, band):
        e = min(T, b0 + band)
        wb = w[b0:e]
        full_row = float(wb.sum())
        suffix = np.cumsum(wb[::-1])[::-1]
        tri_rows = suffix - 0.5 * wb          # row ti in [b0, e): half diagonal + rest
        out.append((b0, e, base, full_row, np.cumsum(tri_rows)))
        wdt = e - b0
        base += b0 * wdt + wdt * (wdt + 1) // 2
    return out


def triangle_range(tile_w, rank: int, world: int, band: int | None = None) -> tuple[int, int]:
    """Balanced contiguous range of the upper-triangular unit space (ti <= tj)
    in the crossing pass's banded order (band width `band` j-tiles; None = one
    band = row-major), where unit (ti, tj) weighs tile_w[tj] (half on the
    diagonal)."""
    import numpy as np

    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    w = np.asarray(tile_w, dtype=np.float64)
    T = len(w)
    U = T * (T + 1) // 2
    W = T if band is None else max(1, int(band))
    bands = _band_unit_weights(w, W)
    band_tot = np.array([b0 * full + (tri[-1] if len(tri) else 0.0)
                         for (b0, e, base, full, tri) in bands])
    band_cum = np.cumsum(band_tot)
    total = float(band_cum[-1]) if len(band_cum) else 0.0

    def unit_at(frac: float) -> int:
        if frac <= 0.0:
            return 0
        if frac >= 1.0:
            return U
        target = frac * total
        k = int(np.searchsorted(band_cum, target, side="left"))
        if k >= len(bands):
            return U
        b0, e, base, full, tri = bands[k]
        t = target - (float(band_cum[k - 1]) if k else 0.0)
        wdt = e - b0
        wb = w[b0:e]
        if b0 > 0 and t <= b0 * full:           # in the full rows below the band
            ti = min(b0 - 1, int(t // full)) if full > 0 else 0
            rem = t - ti * full
            tj_off = int(np.searchsorted(np.cumsum(wb), rem, side="left"))
            return min(U, base + ti * wdt + min(tj_off, wdt - 1) + 1)
        t -= b0 * full
        r = int(np.searchsorted(tri, t, side="left"))
        r = min(r, wdt - 1)
        before = float(tri[r - 1]) if r else 0.0
        within = np.cumsum(np.concatenate(([0.5 * wb[r]], wb[r + 1:])))
        off = int(np.searchsorted(within, t - before, side="left"))
        off = min(off, wdt - r - 1)
        return min(U, base + b0 * wdt + r * wdt - r * (r - 1) // 2 + off + 1)

    return unit_at(rank / world), unit_at((rank + 1) / world)


def triangle_plan(tile_w, world: int, band: int | None = None) -> list[tuple[int, int]]:
    plan = [triangle_range(tile_w, r, world, band) for r in range(world)]
    T = len(tile_w)
    assert plan[0][0] == 0 and plan[-1][1] == T * (T + 1) // 2
    assert all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
    return plan
