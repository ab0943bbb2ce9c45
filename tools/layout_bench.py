"""fr_layout timing: GPU (glr_fr_layout) vs the numpy restatement of the
reference (oracle/glare_oracle.py fr_layout_positions, 1 core) on random
graphs.  python tools/layout_bench.py"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2411_09809_b200 import fr_layout
from paper_2411_09809_b200.configs import random_graph
from oracle.glare_oracle import fr_layout_positions
from paper_2411_09809_b200.model import normalize_edges

for n, m, it, cpu_it in ((4000, 80000, 30, 2), (20000, 40000, 20, 1), (100000, 500000, 10, 0)):
    edges = random_graph(n, m, seed=1)
    fr_layout(edges, iterations=1, seed=1)  # warm
    torch.cuda.synchronize()
    # per-iteration time = (T(1 + it) - T(1)) / it: excludes the host-side
    # preprocessing (normalize_edges, searchsorted, transfers) of each call
    t0 = time.perf_counter(); fr_layout(edges, iterations=1, seed=1); torch.cuda.synchronize()
    t1 = time.perf_counter(); fr_layout(edges, iterations=1 + it, seed=1); torch.cuda.synchronize()
    t2 = time.perf_counter()
    gpu = ((t2 - t1) - (t1 - t0)) / it
    row = {"n": n, "m": m, "iterations": it, "gpu_ms_per_iter": gpu * 1e3,
           "pairs_per_s": n * n / gpu}
    if cpu_it:
        ids = np.unique(edges); ne, _, _ = normalize_edges(edges)
        ei, ej = np.searchsorted(ids, ne[:, 0]), np.searchsorted(ids, ne[:, 1])
        t0 = time.perf_counter(); fr_layout_positions(len(ids), ei, ej, cpu_it, 1, 100.0)
        cpu = (time.perf_counter() - t0) / cpu_it
        row.update({"cpu_ms_per_iter": cpu * 1e3, "speedup": cpu / gpu})
    print(json.dumps(row), flush=True)
