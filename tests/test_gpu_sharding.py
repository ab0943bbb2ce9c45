"""GPU side of the multi-GPU path on one device:

* every rank's interleaved partial equals the oracle's restatement of that
  rank's share (oracle/glare_oracle.py crossing_scan_interleaved), not only
  the sum over ranks;
* the C-ABI combine (glr_allreduce_sum_f64, and the per-rank communicator
  entry points) sums partials with NCCL (world 1 on one GPU);
* two processes build the same strategy="auto" plan: same plan choice, unit
  count and candidate list, so their unit spaces agree (the ranks never
  wait on each other; gloo only compares the plans).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import socket

import numpy as np
import pytest

import cases
from conftest import graph_from, strict_close

pytestmark = pytest.mark.gpu

IDEAL = 7.0 * math.pi / 18.0


@pytest.mark.parametrize("world", [2, 3, 8])
def test_each_rank_matches_oracle_share(gpu, world):
    from oracle import glare_oracle as O
    from paper_2411_09809_b200 import _lib, metrics as M

    g = graph_from(cases.lattice_stress)
    dg = M.DeviceGraph.from_graph(g)
    rec = M.CrossingRecords(dg, "dense", "input")
    tile, band = _lib.lib().glr_crossing_tile(), _lib.lib().glr_crossing_band()
    for r in range(world):
        c, d = rec.partial_interleaved(IDEAL, r, world).tolist()
        oc, od = O.crossing_scan_interleaved(g.xy, g.edges, IDEAL, tile, r, world, band)
        assert int(c) == oc, (world, r)
        assert strict_close(d, od), (world, r)


def test_allreduce_c_abi_single_process(gpu):
    import torch
    from paper_2411_09809_b200 import _lib

    L = _lib.lib()
    buf = torch.tensor([3.0, 0.25, 7.0], dtype=torch.float64, device="cuda:0")
    devs = (ctypes.c_int * 1)(0)
    ptrs = (ctypes.c_void_p * 1)(buf.data_ptr())
    torch.cuda.synchronize()
    rc = L.glr_allreduce_sum_f64(1, devs, ptrs, 3)
    assert rc == 0, L.glr_last_error()
    assert buf.tolist() == [3.0, 0.25, 7.0]  # one rank: the sum is itself
    assert L.glr_allreduce_sum_f64(0, devs, ptrs, 3) == _lib.GLR_EARG


def test_allreduce_c_abi_communicator(gpu):
    import torch
    from paper_2411_09809_b200 import _lib

    L = _lib.lib()
    nbytes = L.glr_nccl_id_bytes()
    assert nbytes == 128
    uid = ctypes.create_string_buffer(nbytes)
    assert L.glr_nccl_unique_id(uid) == 0, L.glr_last_error()
    comm = ctypes.c_void_p()
    assert L.glr_nccl_comm_init(uid, 0, 1, ctypes.byref(comm)) == 0, L.glr_last_error()
    buf = torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    assert L.glr_allreduce_sum_f64_comm(comm, buf.data_ptr(), 2, stream) == 0
    torch.cuda.synchronize()
    assert buf.tolist() == [1.0, 2.0]
    assert L.glr_nccl_comm_destroy(comm) == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


PLAN_GRAPHS = ("C2", "local_lattice", "long_random")


def _plan_graph(name):
    """Graphs above the auto threshold (20k edges): a local lattice takes the
    culled plan, long random edges the dense one, C2 whichever auto picks."""
    from paper_2411_09809_b200 import configs
    from paper_2411_09809_b200.model import LayoutGraph

    if name == "C2":
        return configs.config2()[0]
    rng = np.random.default_rng(5)
    if name == "local_lattice":
        side = 120
        gx, gy = np.meshgrid(np.arange(side, dtype=np.float64), np.arange(side, dtype=np.float64))
        xy = np.stack([gx.ravel(), gy.ravel()], 1) + rng.uniform(-1e-3, 1e-3, (side * side, 2))
        idx = np.arange(side * side).reshape(side, side)
        pairs = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                                np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)])
        return LayoutGraph(np.arange(side * side), xy, pairs)
    n = 8000
    xy = rng.integers(0, 2 ** 16, (n, 2)).astype(np.float64)
    pairs = rng.integers(0, n, (25000, 2))
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    return LayoutGraph(np.arange(n), xy, pairs)


def _plan_worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09809_b200 import metrics as M

        torch.cuda.set_device(0)
        out = {}
        for name in PLAN_GRAPHS:
            g = _plan_graph(name)
            dg = M.DeviceGraph.from_graph(g)
            rec = M.CrossingRecords(dg, "auto", "theta")
            lst = rec.list.cpu().numpy().tobytes() if rec.culled else b""
            part = rec.partial_interleaved(IDEAL, rank, world).tolist()
            out[name] = (rec.culled, rec.units, hashlib.sha256(lst).hexdigest(), part)
        objs = [None] * world
        dist.all_gather_object(objs, out)
        q.put((rank, objs))
    finally:
        dist.destroy_process_group()


def test_two_processes_build_the_same_auto_plan(gpu):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    objs = results[0]
    culled = {name: objs[0][name][0] for name in objs[0]}
    assert culled["local_lattice"] and not culled["long_random"], culled
    for name in objs[0]:
        a, b = objs[0][name], objs[1][name]
        assert a[:3] == b[:3], name  # same plan, unit count and list
        # the two shares add up to the whole
        from oracle import sweep as S

        g = _plan_graph(name)
        c, d = S.crossing_scan(g.xy, g.edges, IDEAL)
        assert int(a[3][0] + b[3][0]) == c
        assert strict_close(a[3][1] + b[3][1], d)


def _big_long_random():
    """Long random edges above the k-d order's threshold (131,072 edges)."""
    from paper_2411_09809_b200.model import LayoutGraph, normalize_edges

    rng = np.random.default_rng(21)
    n, m = 50000, 150000
    xy = rng.integers(0, 2 ** 16, (n, 2)).astype(np.float64)
    pairs = rng.integers(0, n, (m, 2))
    pairs = pairs[np.any(xy[pairs[:, 0]] != xy[pairs[:, 1]], axis=1)]
    e, _, _ = normalize_edges(pairs)
    return LayoutGraph.from_normalized(xy, e)


E2E_GRAPHS = {"local_lattice": lambda: _plan_graph("local_lattice"), "big_long": _big_long_random}


def _e2e_worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09809_b200 import metrics as M, sharding

        torch.cuda.set_device(0)
        out = {}
        for name, make in E2E_GRAPHS.items():
            g = make()
            dg = M.DeviceGraph.from_graph(g)
            for strategy in ("auto", "culled", "dense"):
                # gloo reduces host tensors: combine the device partial on the host
                res = torch.zeros(3, dtype=torch.float64, device="cuda")
                rec = M.CrossingRecords(dg, strategy, "theta",
                                        rows=(rank, world) if strategy != "dense" else None)
                rec.partial_interleaved(IDEAL, rank, world, out=res[0:2])
                host = res.cpu()
                dist.all_reduce(host)
                out[(name, strategy)] = (host.tolist(), rec.culled, rec.rows)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_row_dealt_plans_end_to_end(gpu):
    """Two processes (gloo, one device, never waiting on each other's kernels)
    run the multi-rank path of sharded_evaluate: culled plans dealt by tile
    rows -- with "auto" agreeing through the allreduce of plan costs -- and
    dense interleaved chunks; every strategy's combined result equals the C
    oracle's."""
    import torch.multiprocessing as mp

    from oracle import sweep as S

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_e2e_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, make in E2E_GRAPHS.items():
        g = make()
        c, d = S.crossing_scan(g.xy, g.edges, IDEAL)
        for strategy in ("auto", "culled", "dense"):
            (r0, culled0, rows0), (r1, culled1, rows1) = (results[k][(name, strategy)] for k in (0, 1))
            assert r0 == r1, (name, strategy)               # both ranks hold the sum
            assert culled0 == culled1, (name, strategy)     # ... and took the same plan
            assert int(r0[0]) == c and strict_close(r0[1], d), (name, strategy, r0, c, d)
            if strategy == "culled":
                assert culled0 and rows0 == (0, 2) and rows1 == (1, 2)
