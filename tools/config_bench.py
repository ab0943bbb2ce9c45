"""Per-config timing of all requested metrics (strategy auto), with the
effective pair-test rates.  Used for profiles/rNN_configs.txt.

    python tools/config_bench.py [configs...]
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2411_09809_b200 import configs
from paper_2411_09809_b200 import metrics as M


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return r, best


def run(k):
    t0 = time.perf_counter()
    g, p = configs.make(k)
    gen = time.perf_counter() - t0
    dg = M.DeviceGraph.from_graph(g)
    m, n = g.num_edges, g.num_vertices
    res = {"config": k, "n": n, "m": m, "gen_s": round(gen, 2)}
    for strat in ("auto", "dense") if k != 5 else ("auto", "culled"):
        def cross():
            rec = M.CrossingRecords(dg, strat)
            if os.environ.get("GLR_BENCH_MODE"):  # force a pair-kernel mode (0/1/2)
                rec.set_mode(int(os.environ["GLR_BENCH_MODE"]))
            return rec.partial(p["ideal"], 0, rec.units).tolist(), rec.culled, rec.units

        (out, sec) = timed(cross, reps=1 if (strat == "dense" and k >= 4) else 2)
        (cd, culled, units) = out
        res[f"ec_{strat}"] = {"count": int(cd[0]), "dev": cd[1], "s": sec, "culled": culled,
                              "units": units, "eff_pairs_per_s": m * (m - 1) / 2 / sec}

        def occ():
            plan = M.OcclusionPlan(dg, p["radius"], strat)
            return plan.partial(0, plan.units).item(), plan.culled
        (o, oc), sec = timed(occ)
        res[f"nc_{strat}"] = {"count": int(o), "s": sec, "culled": oc,
                              "eff_pairs_per_s": n * (n - 1) / 2 / sec}
    if "ma" in p["metrics"]:
        _, sec = timed(lambda: M.minimum_angle(dg))
        res["ma_s"] = sec
        _, sec = timed(lambda: M.edge_length_variation(dg))
        res["ml_s"] = sec
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    for k in (sys.argv[1:] or ["1", "2", "3", "4", "5"]):
        run(int(k))
