"""Benchmark: edge-pair crossing tests/s (and node-pair occlusion tests/s) on
BASELINE.json config 5 -- the strong-scaling configuration -- at N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL): every rank builds
the same seeded synthetic C5 graph, owns every world-th chunk of the
upper-triangular tile-pair unit space (crossing; contiguous ranges for
occlusion), and the partials are combined with one allreduce (SURVEY.md
8(e)); scaling is strong (fixed total work).

Step = one fused E_c + E_ca pass (glr_crossing_pairs with the angle sum) over
the whole C5 edge set, inputs resident in HBM (records ~660 MB > 126 MB L2,
so no L2 flush is needed).  `value` = m(m-1)/2 algorithmic edge-pair tests per
second over the K timed steps (max over ranks).  `e2e` = the same metric
through the public API with host (pinned) inputs: H2D of xy+edges, prologue,
pair pass, allreduce, D2H of the result.  `occlusion` = node-pair tests/s of
the N_c pass timed the same way.

`--impl reference` times the reference algorithm on the host CPU instead: the
oracle port (oracle/sweep_oracle.c, the reference's x-sorted crossing scan
restated in C, all host threads) on a bounded sample of the same workload; the
reference itself is pure Python and cannot travel to the GPU box.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG = 5
FP64_PER_PAIR_EC = 18      # DADD/DMUL of the reference predicate
FP64_PER_PAIR_ECA = 22     # + 4 DADD of the fused crossing-angle deviation
FP64_PER_PAIR_NC = 5
# occlusion_filter_kernel hot block (tools/sass_loop.py, 4 j x 8 i = 32 pairs):
# 123 SASS; FMA pipe: 32 FADD2 + 32 FFMA2 = 128 lane-ops
OCC_SASS_PER_PAIR = 123 / 32
OCC_FMA_PER_PAIR = 128 / 32
# The default pair kernel (certified FP32 filter) per pair:
# 8 FFMA + 2 FMUL on the FP32 FMA pipe (issued as packed pairs) and, fused
# with E_ca over theta-ordered edges, 2 DADD on the FP64 pipe (|theta_j -
# (theta_i + s)| and the accumulate; units straddling 0 or pi/2 of theta
# difference, ~1e-4 of them on C5, take 4).
FMA_PER_PAIR = 10
# SASS instructions per pair of the hot block of cross_filter_kernel<angle>
# in classified units with the capped threshold (159 per 16 pairs,
# tools/sass_loop.py / tools/rf_model.py): the issue-slot bound is
# 4 schedulers x 32 lanes x 148 SMs x clock / this.
SASS_PER_PAIR = 159 / 16
# Register-file operand reads per pair of the same block (477 per 16 pairs,
# tools/rf_model.py), and the measured cost of one 32-bit vector-register
# read per scheduler (0.56 cycles: FFMA2 P-S-P 2.75 cycles, FMUL2 P-P 2.2,
# +LEA.HI +1.3, profiles/r02_rfbench.txt).  The model predicts the measured
# per-pair time of the crossing filter (within 2% with the 23% of
# instructions outside the hot block) and of the occlusion filter (3%).
RF_READS_PER_PAIR = 477 / 16
RF_CYCLES_PER_READ = 0.56
OCC_RF_READS_PER_PAIR = 371 / 32
FP64_PER_PAIR_FILTER_ECA = 2
FMA_LANES_PER_CLK_SM = 128   # measured 124 (FFMA2/FMUL2/FADD2, profiles/r01_packed.txt)
FP64_LANES_PER_CLK_SM = 64   # measured 61.7 (profiles/r01_pipes.txt)
# Bytes the pair kernel must read at least once per launch: i-role filter
# record 36 B + j-role record 32 B + theta 8 B per edge.
REC_BYTES_PER_EDGE = 76
CPU_SAMPLE_EDGES = 120_000
CPU_SAMPLE_SEED = 99


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        reasons = [v for k, v in self.NAMES.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def _cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model


def cpu_baseline_sample(g, ideal, threads):
    """Reference algorithm (C port of the x-sorted oracle scan) on a fixed
    random subset of the config's edges, all given host threads."""
    from oracle import sweep as S

    rng = np.random.default_rng(CPU_SAMPLE_SEED)
    m = min(CPU_SAMPLE_EDGES, g.num_edges)
    sub = np.sort(rng.choice(g.num_edges, size=m, replace=False))
    edges = g.edges[sub]
    t0 = time.perf_counter()
    count, dev = S.crossing_scan(g.xy, edges, ideal, threads=threads)
    dt = time.perf_counter() - t0
    pairs = m * (m - 1) / 2
    return pairs / dt, dt, m, count


def run_reference(args, world, rank):
    """--impl reference: the CPU reference algorithm on this box's host."""
    if rank != 0:
        return 0
    from oracle import sweep as S
    from paper_2411_09809_b200 import configs

    g, p = configs.make(CONFIG)
    threads = S.default_threads()
    for _ in range(args.warmup):
        cpu_baseline_sample(g, p["ideal"], threads)
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        v, dt, m, _ = cpu_baseline_sample(g, p["ideal"], threads)
        vals.append(v)
        t_all += dt
    value = args.steps * (CPU_SAMPLE_EDGES * (CPU_SAMPLE_EDGES - 1) / 2) / t_all
    sample = (f"random {CPU_SAMPLE_EDGES}-edge subset of C5 (seed {CPU_SAMPLE_SEED}), "
              f"fused E_c+E_ca x-sorted sweep; pairs counted as m(m-1)/2")
    line = {
        "impl": "reference", "metric": "edge-pair crossing tests/s (E_c+E_ca fused)",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config_desc(g, p, world),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu": _cpu_info()},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _rf_bound(rate, sm_mhz, reads_per_pair):
    peak = 4 * 148 * sm_mhz * 1e6 * 32 / (reads_per_pair * RF_CYCLES_PER_READ)
    return {"reads_per_pair": reads_per_pair, "cycles_per_read": RF_CYCLES_PER_READ,
            "pairs_per_s": peak, "frac": rate / peak,
            "source": "tools/rf_model.py on the hot block; profiles/r02_rfbench.txt"}


def _dram_bytes():
    """DRAM read+write bytes of one full C5 fused launch (ncu), if profiled."""
    path = os.path.join(REPO, "profiles", "r02_dram_c5.txt")
    try:
        with open(path) as f:
            vals = [float(line.split("=")[1].split()[0]) * (1e9 if "Gbyte" in line else 1e6)
                    for line in f if "dram__bytes_" in line and "=" in line]
        return sum(vals) if vals else None
    except (OSError, ValueError, IndexError):
        return None


def _occ_roofline(rate, sm_mhz):
    """Occlusion pass against its two compute ceilings per GPU: the FP32 FMA
    pipe (OCC_FMA_PER_PAIR lane-ops per pair at 128 lanes/clk/SM) and issue
    slots (OCC_SASS_PER_PAIR instructions per pair, 4 schedulers x 32 lanes)."""
    fma_peak = FMA_LANES_PER_CLK_SM * 148 * sm_mhz * 1e6 / OCC_FMA_PER_PAIR
    issue_peak = 4 * 32 * 148 * sm_mhz * 1e6 / OCC_SASS_PER_PAIR
    return {"bound": "fp32-fma", "achieved": rate, "peak": fma_peak, "unit": "pairs/s",
            "frac": rate / fma_peak, "fma_lane_ops_per_pair": OCC_FMA_PER_PAIR,
            "issue_bound": {"sass_per_pair": OCC_SASS_PER_PAIR, "pairs_per_s": issue_peak,
                            "frac": rate / issue_peak},
            "rf_read_bound": _rf_bound(rate, sm_mhz, OCC_RF_READS_PER_PAIR),
            "kernel": "occlusion_filter_kernel"}


def _culled_filter(info, pass_ms, sm_mhz):
    """Pairs the certified filter actually evaluates in the culled pass (the
    blocks neither dropped nor counted whole) against the pass time -- a lower
    bound of cross_filter_kernel's own rate (the pass also runs the full-unit
    kernels, ~8% of it on C5) -- and the FMA-pipe fraction at that rate."""
    if "blocks_filtered" not in info:
        return None
    pairs = info["blocks_filtered"] * info["block_pairs"]
    rate = pairs / (pass_ms * 1e-3)
    peak = FMA_LANES_PER_CLK_SM * 148 * sm_mhz * 1e6
    return {"pairs": pairs, "pairs_per_s": rate, "fma_frac": FMA_PER_PAIR * rate / peak,
            "kernel": "cross_filter_kernel<angle> over the mixed units"}


def _config_desc(g, p, world):
    return {"workload": "C5: Chung-Lu gamma 2.3, 4,000,000 edges / 1,500,000 vertices on the "
                        "2^16 integer lattice (fp64); E_c + E_ca fused pass; N_c at r=8",
            "config_index": CONFIG, "edges": int(g.num_edges), "vertices": int(g.num_vertices),
            "edge_pairs": int(g.num_edges) * (int(g.num_edges) - 1) // 2,
            "node_pairs": int(g.num_vertices) * (int(g.num_vertices) - 1) // 2,
            "ideal_deg": 70.0, "radius": p["radius"], "parallelism": f"units{world}",
            "l2": "inputs (~660 MB records) exceed the 126 MB L2; no flush needed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-layout", action="store_true", help="skip the fr_layout line item")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_2411_09809_b200 import _lib, configs, sharding
    from paper_2411_09809_b200 import metrics as M

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # torchrun (even with one process) exercises the NCCL path end to end
    use_dist = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if use_dist:
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()

    g, p = configs.make(CONFIG)
    ideal, radius = p["ideal"], p["radius"]
    m, n = g.num_edges, g.num_vertices
    P_E = m * (m - 1) / 2
    P_V = n * (n - 1) / 2

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    dg = M.DeviceGraph.from_graph(g, device=dev)
    out = torch.zeros(3, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def crossing_step():
        rec = M.CrossingRecords(dg, order="theta")
        rec.partial_interleaved(ideal, rank, world, out=out[0:2])
        sharding.allreduce_partials(out[0:2])
        del rec  # release before the next step builds its own (allocator reuse)

    def occlusion_step():
        U = M.occlusion_units(n)
        b, e = sharding.shard_range(U, rank, world)
        M.occlusion_partial(dg, M.occlusion_threshold(radius), b, e, out=out[2:3])
        sharding.allreduce_partials(out[2:3])

    # ---- device-resident crossing pass ----
    for _ in range(args.warmup):
        crossing_step()
    barrier()
    L.glr_take_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern_ms = []
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            rec = M.CrossingRecords(dg, order="theta")
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(stream)
            rec.partial_interleaved(ideal, rank, world, out=out[0:2])
            k1.record(stream)
            sharding.allreduce_partials(out[0:2])
            kern_ms.append((k0, k1))
            del rec
        ev1.record(stream)
        barrier()
    launches = int(L.glr_take_launch_count())
    step_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    kernel_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in kern_ms))
    count, dev_sum = out[0:2].tolist()
    value = P_E / (step_ms * 1e-3)

    # ---- occlusion pass ----
    for _ in range(args.warmup):
        occlusion_step()
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        occlusion_step()
    ev1.record(stream)
    barrier()
    occ_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    occ_count = out[2].item()

    # ---- occlusion, culled plan (Morton order + candidate tile pairs) ----
    # wall-clocked: the candidate count is a host sync inside the step
    def occlusion_culled_step():
        plan = M.OcclusionPlan(dg, radius, "culled")
        b, e = sharding.shard_range(plan.units, rank, world)
        plan.partial(b, e, out=out[2:3])
        sharding.allreduce_partials(out[2:3])
        return plan.units

    for _ in range(args.warmup):
        occlusion_culled_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        occ_units = occlusion_culled_step()
    barrier()
    occ_culled_ms = max_over_ranks(1e3 * (time.perf_counter() - t0) / args.steps)
    assert out[2].item() == occ_count, (out[2].item(), occ_count)

    # ---- crossing, culled plan (k-d order + classified tile pairs and
    # blocks; what strategy="auto" runs on C5; tile rows dealt to the ranks
    # for world > 1, as sharded_evaluate does) -- effective rate, same result
    rows = (rank, world) if world > 1 else None
    culled_pass = []

    def crossing_culled_step(stats=False):
        rec = M.CrossingRecords(dg, "culled", rows=rows)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        rec.partial_interleaved(ideal, rank, world, out=out[0:2])
        k1.record(stream)
        sharding.allreduce_partials(out[0:2])
        culled_pass.append((k0, k1))
        # one evaluation at a time, as a caller reading the result sees it (a
        # host running ahead of the pass makes the library's stream-ordered
        # scratch pool grow instead of reusing the previous step's: ~0.26 s once)
        torch.cuda.synchronize()
        info = {"units": rec.units, "mixed": rec.n_mixed, "full": rec.n_full}
        if stats and rec.n_mixed:
            q = L.glr_crossing_sub_quarters()
            nb = (L.glr_crossing_tile() // 128) * q
            sub = rec.sub[:rec.n_mixed].to(torch.int64)
            none = sum(int(((sub >> k) & 1).sum().item()) for k in range(nb))
            fullb = sum(int(((sub >> (nb + k)) & 1).sum().item()) for k in range(nb))
            info.update(blocks_per_unit=nb, block_pairs=128 * (L.glr_crossing_tile() // q),
                        blocks_none=none, blocks_full=fullb,
                        blocks_filtered=nb * rec.n_mixed - none - fullb)
        del rec
        return info

    for _ in range(min(args.warmup, 1)):
        crossing_culled_step()
    barrier()
    torch.cuda.synchronize()
    culled_pass.clear()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cross_info = crossing_culled_step()
    torch.cuda.synchronize()
    barrier()
    cross_culled_ms = max_over_ranks(1e3 * (time.perf_counter() - t0) / args.steps)
    cross_pass_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in culled_pass))
    assert out[0].item() == count, (out[0].item(), count)
    cross_info = crossing_culled_step(stats=True)  # block statistics, untimed
    cross_units = (cross_info["units"], cross_info["mixed"], cross_info["full"])

    # ---- fr_layout: repulsion pairs/s, rank 0 ----
    layout = None
    if rank == 0 and not args.no_layout:
        from paper_2411_09809_b200 import fr_layout
        from paper_2411_09809_b200.configs import random_graph

        ln, lm, lit = 20000, 40000, 20
        ledges = random_graph(ln, lm, seed=1)
        fr_layout(ledges, iterations=1, seed=1)
        torch.cuda.synchronize()
        # per-iteration device time: (T(1 + lit) - T(1)) / lit, which removes
        # the per-call host preprocessing (normalize_edges, transfers)
        t0 = time.perf_counter()
        fr_layout(ledges, iterations=1, seed=1)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        fr_layout(ledges, iterations=1 + lit, seed=1)
        torch.cuda.synchronize()
        lay_s = ((time.perf_counter() - t1) - (t1 - t0)) / lit
        layout = {"metric": "fr_layout repulsion pair terms/s (bit-exact with the reference)",
                  "value": ln * ln / lay_s, "unit": "pairs/s",
                  "ms_per_iteration": lay_s * 1e3,
                  "config": {"vertices": ln, "edges": lm, "iterations": lit,
                             "graph": "random_graph(20000, 40000, seed=1)"}}

    # ---- end-to-end through the public API with pinned host inputs ----
    xy_h = torch.from_numpy(g.xy).pin_memory()
    ed_h = torch.from_numpy(g.edges).pin_memory()
    h2d = xy_h.numel() * 8 + ed_h.numel() * 8
    e2e_times = []
    for i in range(args.e2e_steps + 1):
        barrier()
        t0 = time.perf_counter()
        dge = M.DeviceGraph(xy_h.to(dev, non_blocking=True), ed_h.to(dev, non_blocking=True))
        # the public API's default strategy ("auto": the culled plan on C5)
        res = sharding.sharded_evaluate(dge, None, ideal, rank, world, strategy="auto")
        c_e2e, d_e2e, _ = res.tolist()  # D2H of the step's result
        dt = time.perf_counter() - t0
        if i > 0:  # first iteration warms the pinned-copy path
            e2e_times.append(dt)
        assert c_e2e == count, (c_e2e, count)
    e2e_ms = max_over_ranks(1e3 * statistics.mean(e2e_times))
    e2e_value = P_E / (e2e_ms * 1e-3)

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return 0

    # Roofline of the dominant kernel (cross_filter_kernel<angle>): its
    # algorithm loads the FP32 FMA pipe most (10 lane-ops per pair against
    # 128 lanes/clk/SM, vs 4 FP64 lane-ops against 64), so that pipe bounds it.
    clk = clocks.summary()
    recs = M.CrossingRecords(dg, order="theta")
    fast, mode = recs.fast_path(), recs.mode()
    pairs_per_launch = P_E / world
    pair_rate = pairs_per_launch / (kernel_ms * 1e-3)
    sm_mhz = clk.get("sm_mhz") or 1965.0
    peak_run = FMA_LANES_PER_CLK_SM * 148 * sm_mhz * 1e6 / 1e12
    peak_max = FMA_LANES_PER_CLK_SM * 148 * 1965e6 / 1e12
    achieved = FMA_PER_PAIR * pair_rate / 1e12
    fp64_peak_run = FP64_LANES_PER_CLK_SM * 148 * sm_mhz * 1e6 / 1e12
    cpu = None  # the CPU reference sample runs on rank 0 at N=1 only
    if not args.no_cpu_baseline and world == 1:
        from oracle import sweep as S

        threads = S.default_threads()
        v, dt, ms_, _ = cpu_baseline_sample(g, ideal, threads)
        cpu = {"value": v, "unit": "pairs/s", "cores": threads, "kind": "port",
               "sample": f"random {ms_}-edge subset of C5, fused E_c+E_ca x-sorted sweep "
                         f"(oracle/sweep_oracle.c), {dt:.1f} s",
               "cpu": _cpu_info()}
    line = {
        "metric": "edge-pair crossing tests/s (E_c+E_ca fused)",
        "value": value,
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": _config_desc(g, p, world),
        "result": {"edge_crossing": int(count), "dev_sum": dev_sum,
                   "edge_crossing_angle": 1.0 - (dev_sum / ideal) / count if count else 1.0,
                   "node_occlusion": int(occ_count), "fast_window": fast},
        "occlusion": {"metric": "node-pair occlusion tests/s", "value": P_V / (occ_ms * 1e-3),
                      "unit": "pairs/s", "ms_per_step": occ_ms, "strategy": "dense",
                      "kernel": "occlusion_filter_kernel (certified packed-FP32 filter, "
                                "FP64 re-test of near-threshold pairs)",
                      # the reference formulation (5 FP64 per pair) at this
                      # rate against the FP64 peak (> 1: the filter does not
                      # execute it for most pairs)
                      "fp64_equivalent": {
                          "fp64_per_pair": FP64_PER_PAIR_NC,
                          "tflops": FP64_PER_PAIR_NC * P_V / world / (occ_ms * 1e-3) / 1e12,
                          "vs_fp64_peak_at_max_clock": FP64_PER_PAIR_NC * P_V / world
                          / (occ_ms * 1e-3) / (64 * 148 * 1965e6)},
                      "roofline": _occ_roofline(P_V / world / (occ_ms * 1e-3), sm_mhz),
                      "culled": {"value": P_V / (occ_culled_ms * 1e-3), "unit": "pairs/s",
                                 "ms_per_step": occ_culled_ms, "candidate_units": occ_units,
                                 "dense_units": M.occlusion_units(n),
                                 "note": "effective rate: same count, Morton order + "
                                         "candidate tile pairs (incl. plan build)"}},
        "crossing_culled": {"metric": "edge-pair crossing tests/s (E_c+E_ca fused), culled plan",
                            "value": P_E / (cross_culled_ms * 1e-3), "unit": "pairs/s",
                            "ms_per_step": cross_culled_ms, "pass_ms": cross_pass_ms,
                            "candidate_units": cross_units[0],
                            "mixed_units": cross_units[1], "full_units": cross_units[2],
                            "dense_units": M.crossing_units(m),
                            "blocks": {k: v for k, v in cross_info.items()
                                       if k.startswith("block")},
                            "filter": _culled_filter(cross_info, cross_pass_ms, sm_mhz),
                            "note": "effective rate (m(m-1)/2 / time): same count and sum, "
                                    "(orientation, k-d tree over the endpoints) order + "
                                    "classified tile pairs and slice x quarter blocks -- "
                                    "certified-empty ones dropped, certified-full ones counted "
                                    "without a predicate (incl. plan build); the public API's "
                                    "strategy='auto' on C5; this rank's tile rows for N > 1"},
        "layout": layout,
        "roofline": {"bound": "fp32-fma", "achieved": achieved, "peak": peak_run,
                     "unit": "T lane-op/s (FP32 FFMA/FMUL on the FMA pipe)",
                     "frac": achieved / peak_run,
                     "frac_at_max_clock": achieved / peak_max, "peak_at_max_clock": peak_max,
                     "peak_source": "128 FP32 lanes/clk/SM x 148 SMs x median SM clock under "
                                    "load (microbenchmarked FFMA2/FMUL2/FADD2: 124 "
                                    "lanes/clk/SM, profiles/r01_packed.txt)",
                     "kernel": "cross_filter_kernel<angle>" if mode == 2 else
                               "cross_pairs_kernel<mode %d>" % mode,
                     "pair_kernel_mode": mode,
                     "kernel_ms": kernel_ms,
                     "ops_per_pair": {"fp32_fma_pipe": FMA_PER_PAIR,
                                      "fp64_pipe": FP64_PER_PAIR_FILTER_ECA},
                     "fp64_pipe_frac": FP64_PER_PAIR_FILTER_ECA * pair_rate / 1e12 / fp64_peak_run,
                     # the reference formulation (22 FP64
                     # instructions per pair) at this pair rate, against the
                     # FP64 peak: > 1 because the filter retires most pairs
                     # without FP64 arithmetic
                     "fp64_equivalent": {"fp64_per_pair": FP64_PER_PAIR_ECA,
                                         "tflops": FP64_PER_PAIR_ECA * pair_rate / 1e12,
                                         "vs_fp64_peak": FP64_PER_PAIR_ECA * pair_rate / 1e12
                                         / fp64_peak_run},
                     # DRAM read+write bytes of one full-C5 launch from ncu
                     # (profiles/r01_dram_c5_filter.txt); per-rank share for N>1.
                     "traffic": (_dram_bytes() / world) if _dram_bytes() else None,
                     "traffic_unit": "bytes/launch (dram__bytes_read+write, ncu)",
                     "issue_bound": {"sass_per_pair": SASS_PER_PAIR,
                                     "pairs_per_s": 4 * 32 * 148 * sm_mhz * 1e6 / SASS_PER_PAIR,
                                     "frac": pair_rate / (4 * 32 * 148 * sm_mhz * 1e6
                                                          / SASS_PER_PAIR)},
                     # the resource that binds (K2): register-file
                     # operand reads, RF_CYCLES_PER_READ scheduler cycles each
                     "rf_read_bound": _rf_bound(pair_rate, sm_mhz, RF_READS_PER_PAIR),
                     "algorithmic_bytes": REC_BYTES_PER_EDGE * m},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "pairs/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 3 * 8,
                "strategy": "auto: what edge_crossing_angle(g) runs -- on C5 the culled plan "
                            "(k-d order, classified tile pairs and blocks; plan build "
                            "included); the line's top-level value is the dense "
                            "theta-ordered pass, device-resident"},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
