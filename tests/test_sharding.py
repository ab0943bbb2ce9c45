"""Multi-rank path on CPU: world-size-2 gloo process group running the same
ownership rules and allreduce code the NCCL ranks run (paper_2411_09809_b200/
sharding.py): interleaved chunk ownership of the crossing units (the rule
production uses, crossing.cu chunk_for, restated in oracle/glare_oracle.py
and checked against the library's glr_crossing_chunk here) and contiguous
ranges of the occlusion units.  Per-rank partials come from the oracle's
unit-range restatement (the CUDA kernels' contract, checked against them in
tests/test_gpu_parity.py)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_09809_b200 import sharding

IDEAL = 7.0 * np.pi / 18.0
TILE_E = 256   # glr_crossing_tile()
BAND = 2048    # glr_crossing_band()
TILE_V = 1024


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import cases
        from conftest import graph_from
        from oracle import glare_oracle as O

        g = graph_from(cases.lattice_stress)
        Tv = -(-g.num_vertices // TILE_V)
        c, d = O.crossing_scan_interleaved(g.xy, g.edges, IDEAL, TILE_E, rank, world, BAND)
        bv, ev = sharding.shard_range(Tv * (Tv + 1) // 2, rank, world)
        occ = O.node_occlusion_units(g.xy, 1.0, TILE_V, bv, ev)
        buf = torch.tensor([float(c), d, float(occ)], dtype=torch.float64)
        sharding.allreduce_partials(buf)
        q.put((rank, buf.tolist()))
    finally:
        dist.destroy_process_group()


def test_shard_plan_tiles_unit_space():
    for U in (1, 2, 7, 55, 30_517_578):
        for world in (1, 2, 4, 8):
            plan = sharding.shard_plan(U, world)
            assert sum(e - b for b, e in plan) == U
            sizes = [e - b for b, e in plan]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.shard_range(10, 2, 2)


def test_gloo_world2_partials_sum_to_oracle():
    import cases
    from conftest import graph_from
    from oracle import glare_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = graph_from(cases.lattice_stress)
    c, d = O.crossing_scan(g.xy, g.edges, IDEAL)
    occ = O.node_occlusion(g.xy, 1.0)
    for rank in (0, 1):
        rc, rd, ro = results[rank]
        assert rc == c == 4194903
        assert abs(rd - d) <= 1e-9 * abs(d)
        assert ro == occ == 9588


def _rows_worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import cases
        from conftest import graph_from
        from oracle import glare_oracle as O
        from paper_2411_09809_b200 import metrics as M

        g = graph_from(cases.lattice_stress)
        # row ownership of the culled plan (32-edge tiles: 188 rows to deal)
        c, d = O.crossing_scan_rows(g.xy, g.edges, IDEAL, 32, rank, world)
        buf = torch.tensor([float(c), d, 0.0], dtype=torch.float64)
        sharding.allreduce_partials(buf)
        # the ranks' agreement on "auto": the summed plan cost is the same everywhere
        cost = M._global_cost(100.0 + rank, world, torch.device("cpu"))
        q.put((rank, buf.tolist(), cost))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_row_ownership_sums_to_oracle():
    """Culled plans deal tile ROWS to the ranks (sharding.sharded_evaluate,
    glr_crossing_candidates_rows): the oracle's restatement of that rule over
    two gloo ranks gives the whole result, and both ranks see one plan cost."""
    import cases
    from conftest import graph_from
    from oracle import glare_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {r: (b, c) for r, b, c in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = graph_from(cases.lattice_stress)
    c, d = O.crossing_scan(g.xy, g.edges, IDEAL)
    for rank in (0, 1):
        (rc, rd, _), cost = results[rank]
        assert rc == c == 4194903
        assert abs(rd - d) <= 1e-9 * abs(d)
        assert cost == 201.0


def test_row_ownership_partitions_the_triangle():
    from oracle import glare_oracle as O

    rng = np.random.default_rng(4)
    xy = rng.integers(0, 64, (300, 2)).astype(np.float64)
    e = rng.integers(0, 300, (700, 2))
    e = e[np.any(xy[e[:, 0]] != xy[e[:, 1]], axis=1)]
    want = O.crossing_scan(xy, e, IDEAL)
    for world in (1, 2, 3, 8):
        parts = [O.crossing_scan_rows(xy, e, IDEAL, 64, r, world) for r in range(world)]
        assert sum(p[0] for p in parts) == want[0]
        assert abs(sum(p[1] for p in parts) - want[1]) <= 1e-9 * want[1]


def test_balanced_triangle_and_weighted_ranges():
    rng = np.random.default_rng(0)
    for T in (1, 2, 7, 60):
        w = rng.uniform(0.5, 2.0, T)
        from oracle.glare_oracle import _band_coords

        for band in (None, 1, 3, 16):
            W = T if band is None else band
            U = T * (T + 1) // 2
            order = [_band_coords(u, T, W) for u in range(U)]
            unit_w = np.array([w[tj] * (0.5 if ti == tj else 1.0) for ti, tj in order])
            for world in (1, 2, 3, 8):
                plan = sharding.triangle_plan(w, world, band)
                # per-rank weight is balanced within one unit's weight
                loads = [unit_w[b:e].sum() for b, e in plan]
                assert max(loads) - min(loads) <= 2.0 * unit_w.max() + 1e-9, (T, band, world)
        lst_w = rng.uniform(0.5, 2.0, 50)
        cuts = [sharding.weighted_range(lst_w, r, 4) for r in range(4)]
        assert cuts[0][0] == 0 and cuts[-1][1] == 50
        assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))


def test_interleaved_chunk_matches_library():
    """The oracle's restatement of the chunk rule equals the library's
    (glr_crossing_chunk: host code, no GPU needed), and chunks of every rank
    tile the unit space exactly once."""
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib

    lib = _lib.host_lib()
    assert lib.glr_crossing_tile() == TILE_E and lib.glr_crossing_band() == BAND
    rng = np.random.default_rng(1)
    spans = [1, 2, 591, 592, 593, 4735, 4736, 9473, 122_078_125, 66_337_020, 2 ** 40]
    spans += [int(x) for x in rng.integers(1, 10 ** 9, 40)]
    for span in spans:
        for world in (1, 2, 3, 4, 7, 8, 16):
            assert lib.glr_crossing_chunk(span, world) == O.interleaved_chunk(span, world)
    for span in (1, 7, 300, 5000, 70_001):
        for world in (1, 2, 3, 8):
            chunk = O.interleaved_chunk(span, world)
            owners = [O.interleaved_owner(u, 0, chunk, world) for u in range(span)]
            counts = np.bincount(owners, minlength=world)
            assert counts.sum() == span
            assert counts.max() - counts.min() <= chunk
