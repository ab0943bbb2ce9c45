"""Edge orders for the classified culled plan, tried on the host: the edges
are permuted in numpy, handed to the library in that order (no device sort),
and the classified plan + fused pass are timed and checked against the C5
golden.
    python tools/kd_order_probe.py [variant ...]
variants: lib (the library's own order), lib-morton, kd-cycle, kd-extent[-nogrp][-leafN][-hubN]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_09809_b200 import configs, metrics as M  # noqa: E402

TILE = 256
HUB = 16384
LEAF = 64


def pq(xy, edges):
    a, b = xy[edges[:, 0]], xy[edges[:, 1]]
    pa = (a[:, 0] < b[:, 0]) | ((a[:, 0] == b[:, 0]) & (a[:, 1] <= b[:, 1]))
    P = np.where(pa[:, None], a, b)
    Q = np.where(pa[:, None], b, a)
    return np.concatenate([P, Q], axis=1)  # px py qx qy


def kd_order(xy, edges, rule, groups=True, hub=HUB, theta_w=0.0):
    m = len(edges)
    c = pq(xy, edges)
    ext = c.max(axis=0) - c.min(axis=0)
    ext[ext == 0] = 1.0
    cn = (c - c.min(axis=0)) / ext
    if theta_w > 0:  # a fifth coordinate: the direction, weighted
        th = np.mod(np.arctan2(c[:, 3] - c[:, 1], c[:, 2] - c[:, 0]), np.pi) / np.pi
        cn = np.concatenate([cn, theta_w * th[:, None]], axis=1)
    up = ((c[:, 2] - c[:, 0]) * (c[:, 3] - c[:, 1]) >= 0).astype(np.int64)
    deg = np.bincount(edges.ravel(), minlength=len(xy))
    du, dv = deg[edges[:, 0]], deg[edges[:, 1]]
    hubv = np.where(du >= dv, edges[:, 0], edges[:, 1])
    grp = np.where(np.maximum(du, dv) >= hub, hubv + 1, 0) if groups else np.zeros(m, np.int64)
    top = grp * 2 + up
    perm = np.argsort(top, kind="stable")
    tops = top[perm]
    bounds = np.flatnonzero(np.diff(tops)) + 1
    segs = list(zip(np.r_[0, bounds], np.r_[bounds, m]))
    # recursion on position ranges, splits at tile boundaries
    stack = [(int(s), int(e), 0) for s, e in segs]
    while stack:
        s, e, lvl = stack.pop()
        b = None
        for al in (TILE, 128, 64, 32, 16):
            if al < LEAF:
                break
            lo = s // al + 1          # first boundary index with lo*al > s
            hi = (e - 1) // al        # last boundary index with hi*al < e
            if lo <= hi:
                mid = (s + e) / 2
                b = int(min(max(round(mid / al), lo), hi)) * al
                break
        if b is None:
            continue
        idx = perm[s:e]
        if rule == "cycle":
            d = lvl % 4
        else:
            sub = cn[idx]
            d = int(np.argmax(sub.max(axis=0) - sub.min(axis=0)))
        k = b - s
        part = np.argpartition(cn[idx, d], k - 1 if k > 0 else 0)
        perm[s:e] = idx[part]
        stack.append((s, b, lvl + 1))
        stack.append((b, e, lvl + 1))
    return perm


def run(dg, g, p, es, want, label, reps=2):
    for r in range(reps):
        rec = M.CrossingRecords.__new__(M.CrossingRecords)
        rec.m, rec.n = dg.num_edges, dg.num_vertices
        rec.list = rec.sub = rec.rows = None
        torch.cuda.synchronize()
        t = time.perf_counter()
        rec._prepare(dg.xy, es)
        rec.list, rec.sub, rec.n_mixed, rec.n_full = M._classified_candidates(rec.buf, rec.n, rec.m)
        torch.cuda.synchronize()
        build = time.perf_counter() - t
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        c, d = rec.partial_interleaved(p["ideal"], 0, 1).tolist()
        b.record()
        torch.cuda.synchronize()
        fused = a.elapsed_time(b)
        a.record()
        c0 = rec.partial_interleaved(None, 0, 1)[0].item()
        b.record()
        torch.cuda.synchronize()
        ec = a.elapsed_time(b)
        from paper_2411_09809_b200 import _lib
        nbk = 2 * _lib.lib().glr_crossing_sub_quarters()
        sub = rec.sub[:rec.n_mixed].to(torch.int64)
        bits = sum(int(((sub >> k) & 1).sum().item()) for k in range(nbk))
        fbits = sum(int(((sub >> (nbk + k)) & 1).sum().item()) for k in range(nbk))
        dec = (sub | (sub >> nbk)) & ((1 << nbk) - 1)
        act = torch.zeros_like(dec)
        for k in range(nbk):
            act += 1 - ((dec >> k) & 1)
        hist = torch.bincount(act, minlength=nbk + 1).tolist()
        ok = int(c) == want["ec"] and int(c0) == want["ec"] and abs(d - want["dev"]) <= 1e-9 * want["dev"]
        print(json.dumps({"order": label, "rep": r, "prep_class_ms": round(build * 1e3, 1),
                          "fused_ms": round(fused, 1), "ec_ms": round(ec, 1), "mixed": rec.n_mixed,
                          "full": rec.n_full, "sub_none": bits, "sub_full": fbits, "sub_blocks": nbk * rec.n_mixed, "active_blocks_hist": hist,
                          "dense_units": M.crossing_units(g.num_edges), "golden_ok": ok}), flush=True)
        del rec


def main():
    variants = sys.argv[1:] or ["lib", "kd-cycle", "kd-extent"]
    want = json.load(open("tests/golden/golden.json"))["configs"]["C5"]
    g, p = configs.config5()
    dg = M.DeviceGraph.from_graph(g)
    for v in variants:
        if v.startswith("lib"):
            from paper_2411_09809_b200 import _lib
            _lib.lib().glr_spatial_set_kd(0 if "morton" in v else 1)
            es = torch.empty_like(dg.edges)
            for _ in range(2):
                torch.cuda.synchronize()
                t = time.perf_counter()
                _lib.check(_lib.lib().glr_spatial_sort_edges(M._ptr(dg.xy), dg.num_vertices,
                                                             M._ptr(dg.edges), dg.num_edges,
                                                             M._ptr(es), M._stream()), "sort")
                torch.cuda.synchronize()
                print(v, "device sort ms", round(1e3 * (time.perf_counter() - t), 2), flush=True)
        else:
            t = time.perf_counter()
            import re
            global LEAF
            mleaf, mhub = re.search(r"leaf(\d+)", v), re.search(r"hub(\d+)", v)
            mth = re.search(r"theta([0-9.]+)", v)
            LEAF = int(mleaf.group(1)) if mleaf else 64
            perm = kd_order(g.xy, g.edges, "cycle" if "cycle" in v else "extent",
                            groups="nogrp" not in v, hub=int(mhub.group(1)) if mhub else HUB,
                            theta_w=float(mth.group(1)) if mth else 0.0)
            print(v, "host order s", round(time.perf_counter() - t, 1), flush=True)
            es = torch.from_numpy(np.ascontiguousarray(g.edges[perm])).to(dg.edges.device)
        run(dg, g, p, es, want, v)


if __name__ == "__main__":
    main()
