#!/usr/bin/env python
"""Benchmark: enhanced-DPSO particle-iterations/s at N=1000 viewpoints.

One "step" = one generation of the whole swarm (update -> mutation every
3rd generation -> gbest select -> 2-opt when gbest stalled -> finalize),
i.e. P particle-iterations, on synthetic input resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c4|c5]

Default workload = BASELINE.json configs[1] (the metric's N=1000 case):
random-Euclidean N=1000 extended TSP (conftest.py:27-31 generator,
default_rng(1000)), swarm P=1024, paper defaults (w=1, phi1=phi2=0.4,
mutation every 3 gens, 2-opt on stall), numpy-exact PCG64 streams.

Timing: W untimed warm-up generations, then K generations each bracketed by
CUDA events on the launching stream, with an L2 flush (256 MiB write)
between timed generations, outside the events; barrier + synchronize around
the timed region; max over ranks.  Multi-GPU: island model (one swarm per
rank, gbest exchanged over NCCL every --exchange-every generations;
"scaling": "weak").  ``--impl reference`` times the oracle port of the
reference CPU algorithm (oracle/dpso_oracle.py) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-iterations/sec at N=1000 viewpoints"
UNIT = "particle-iterations/s"

CONFIGS = {
    "c1": dict(n=15, P=32, G=100, matrix="wall",
               workload="C1: pkg/scenes/wall.json (N=15) via the reference "
                        "pipeline, P=32, G=100, boustrophedon seed"),
    "c2": dict(n=1000, P=1024, G=500, matrix="euclid",
               workload="C2: synthetic N=1000 extended TSP (random Euclidean,"
                        " default_rng(1000)), swarm P=1024, 500-generation "
                        "schedule, enhanced DPSO (paper defaults)"),
    "c2i": dict(n=1000, P=1024, G=500, matrix="euclid_int",
                workload="C2 with integer costs: floor(1000 x random-Euclidean "
                         "N=1000), swarm P=1024 (scene-like integer matrix)"),
    "c3": dict(n=500, P=16384, G=100, matrix="grid",
               workload="C3: bridge-sized synthetic instance N=500 (integer "
                        "grid costs, many ties), swarm P=16384"),
    "c2s": dict(n=816, P=1024, G=500, matrix="scene:office",
                workload="C2 scene-shaped: synthetic office floor (100x48x32"
                         " voxels, walls, pillars, partition, desks), 816 "
                         "viewpoints, obstacle-aware costs from the device "
                         "cost build (graph.py:41-78 semantics), swarm "
                         "P=1024"),
    "c3s": dict(n=500, P=16384, G=100, matrix="scene:bridge",
                workload="C3 scene-shaped: synthetic girder bridge with "
                         "dense clutter (120x40x30 voxels), 500 viewpoints "
                         "at 1-3 voxels standoff, axis weights (1,1,2), "
                         "device cost build, swarm P=16384, 2-opt every "
                         "stalled generation"),
    "c4": dict(n=2000, P=65536, G=50, matrix="euclid",
               workload="C4: synthetic N=2000 extended TSP, P=65536"),
    "c5": dict(n=10000, P=65536, G=20, matrix="euclid", ee=False,
               rng="philox",
               workload="C5: synthetic N=10000, P=65536 per GPU, islands, "
                        "use_edge_exchange=False, Philox production RNG"),
}


SCENE_META = {}


def make_matrix(cfg):
    import numpy as np
    n = cfg["n"]
    if cfg["matrix"].startswith("scene:"):
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import scenes
        t0 = time.perf_counter()
        cost, virt, vcost, meta = scenes.scene_matrix(cfg["matrix"][6:])
        meta["cost_build_wall_s"] = time.perf_counter() - t0
        meta["virtual_pairs"] = int(virt.sum() // 2)
        SCENE_META.update(meta)
        return cost, None
    if cfg["matrix"] == "wall":
        with open(os.path.join(ROOT, "tests", "golden",
                               "golden_e2e.json")) as fh:
            g = json.load(fh)
        return np.array(g["matrices"]["wall"], dtype=float), \
            g["seed_tours"]["wall"]
    rng = np.random.default_rng(1000)
    if cfg["matrix"] == "grid":
        side = int(math.ceil(math.sqrt(n)))
        idx = np.arange(n)
        pts = np.stack([idx % side, idx // side], 1).astype(float)
        d = np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)
        return d, None
    pts = rng.random((n, 2)) * 10.0
    c = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(c, 0.0)
    if cfg["matrix"] == "euclid_int":
        c = np.floor(c * 1000.0)
    return c, None


RNG = "numpy"


def solver_params(cfg, P, G, seed):
    p = dict(n_particles=P, max_generations=G, stall_generations=G,
             use_edge_exchange=cfg.get("ee", True), random_state=seed)
    return p


def gpu_params(cfg, P, G, seed):
    p = solver_params(cfg, P, G, seed)
    p["rng"] = RNG
    return p


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,"
              "clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        import threading
        self.lines = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return self
        first = threading.Event()

        def pump():
            for line in self.proc.stdout:
                self.lines.append(line)
                first.set()
        self.thread = threading.Thread(target=pump, daemon=True)
        self.thread.start()
        first.wait(timeout=10.0)  # sampler is live before the timed region
        self.skip = len(self.lines)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=5)
            self.out = "".join(self.lines[self.skip:])

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap")
        reasons = sorted({names[i] for _, _, fl in rows
                          for i, f in enumerate(fl) if f.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ cpu baseline
def cpu_sample(cost, cfg, P_cpu=32, budget_s=10.0, max_gens=400, warm=1,
               seed=0, seed_tour=None):
    """Oracle port of the reference (single thread) on a bounded sample:
    P_cpu particles of the same matrix; returns (rate, gens, seconds)."""
    from oracle.dpso_oracle import OracleSolver
    s = OracleSolver(**solver_params(cfg, P_cpu, 10 ** 6, seed),
                     seed_tour=seed_tour)
    s.start(cost)
    for _ in range(warm):
        s.generation()
    t0 = time.perf_counter()
    g = 0
    while g < max_gens:
        s.generation()
        g += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return P_cpu * g / dt, g, dt


def _ref_worker(args):
    cfg_name, steps, warmup, seed = args
    cfg = CONFIGS[cfg_name]
    cost, seed_tour = make_matrix(cfg)
    from oracle.dpso_oracle import OracleSolver
    s = OracleSolver(**solver_params(cfg, 32, 10 ** 6, seed),
                     seed_tour=seed_tour)
    s.start(cost)
    for _ in range(warmup):
        s.generation()
    t0 = time.perf_counter()
    for _ in range(steps):
        s.generation()
    return 32 * steps, time.perf_counter() - t0


def run_reference(args, cfg_name, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    steps = args.steps
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_ref_worker, [(cfg_name, steps, args.warmup, 100 + i)
                                     for i in range(cores)])
    wall = time.perf_counter() - t0
    work = sum(r[0] for r in res)
    tmax = max(r[1] for r in res)
    value = work / tmax
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tmax / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(cfg_name, cfg, args,
                              int(os.environ.get("WORLD_SIZE", args.gpus))),
        "cpu_baseline": {
            "value": value, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{cores} concurrent processes of the oracle port "
                       f"(oracle/dpso_oracle.py, single-threaded Python+numpy"
                       f" like the reference), each a 32-particle swarm on "
                       f"the same matrix, {args.warmup} warm-up + {steps} "
                       f"timed generations; one step = one generation of "
                       f"each 32-particle sample (wall {wall:.1f}s)")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    # the port against the unmodified reference solver, measured in the
    # build container (tools/port_vs_reference.py): same results, same speed
    try:
        with open(os.path.join(ROOT, "profiles", "r02",
                               "port_vs_reference.json")) as fh:
            pv = json.load(fh)
        line["cpu_baseline"]["port_vs_reference"] = {
            k: pv[k] for k in ("n", "P", "generations", "identical",
                               "reference_rate", "port_rate", "unit")}
    except Exception:
        pass
    print(json.dumps(line), flush=True)


def config_dict(cfg_name, cfg, args, world=1):
    return {"workload": cfg["workload"], "config": cfg_name, "n": cfg["n"],
            "particles_per_gpu": cfg["P"], "global_particles":
                cfg["P"] * world,
            "generation_schedule": cfg["G"],
            "parallelism": f"islands{world}" if world > 1 else "1gpu",
            "exchange_every": args.exchange_every if world > 1 else None,
            "rng": {"numpy": "numpy-pcg64-exact",
                    "philox": "philox4x32-10"}[RNG],
            "l2": "flushed between timed steps (256 MiB write)",
            **({"scene": dict(SCENE_META)} if SCENE_META else {})}


# --------------------------------------------------------------- our arm
def band_kernels(cfg, band):
    """Kernels of one band-scan launch: column records + scan (+ the FILTER
    overflow re-scan)."""
    exact = (band == 1 if band else
             cfg["matrix"] in ("grid", "euclid_int", "wall"))
    return (2 if band else 1) + (0 if exact else 1)


def kernels_per_generation(cfg, band=0, bound=0):
    """(kernels every generation's CUDA graph launches, extra kernels of a
    mutating generation).  Generations with gen % mutation_period != 0 run
    a graph without the mutation call; device flags make kernels a
    generation does not need (the 2-opt scan when gbest improved, ...) exit
    at entry, but they still launch.  band: dpso_scan_band (1/2: the band
    scan and its column-record kernel).  bound: the bounded scan runs
    first; the band scan launches after it every pass (it exits at once
    when the bounded scan hands it no particle), without its column-record
    kernel."""
    k = 1 + 1 + 1  # gen_begin, update, fitness (with the pbest copy)
    k += 1         # select
    if cfg.get("ee", True):
        # scan kernels (bounded scan, or the band / column scan), apply,
        # finalize
        # with the bounded scan: bounded scan + band scan (the bounded scan
        # writes the column records of the particles it hands over, and the
        # apply re-scans a FILTER overflow itself)
        k += 2 if bound else band_kernels(cfg, band)
        k += 2
    # mutation: hash, rank, dedupe, verify, lists, copy (P <= 1024: rank,
    # dedupe, verify and lists in one single-CTA kernel)
    m = 3 if cfg["P"] <= 1024 else 6
    if RNG == "philox":
        m += 1     # Philox sampler
    else:
        m += 2 + 2  # sampler + fix; stream gen + walk (forked stream)
    m += 1 + 1     # swap, then fitness (+ pbest copy) of the mutated
    return k, m


def gpu_launch_count(cfg, first_gen, gens, period=3, band=0, bound=0):
    base, mut = kernels_per_generation(cfg, band, bound)
    n_mut = sum(1 for g in range(first_gen, first_gen + gens)
                if g % period == 0)
    return base * gens + mut * n_mut


def scan_floors(cost, params, seed_body, n_seed, P, gens=6, band=0):
    """The scan's own floor, live: the same launch reduced to its row stream
    (band scan: DPSO_BAND_PROBE=1; column scan: DPSO_SCAN_STREAM_ONLY=1,
    and =2 for the stream plus every pair's gathers)."""
    import numpy as np
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    from paper_1706_04399_b200.solver import numpy_stream_states
    out = {}
    probes = ((("stream_only_ms", "DPSO_BAND_PROBE", "1"),) if band else
              (("stream_only_ms", "DPSO_SCAN_STREAM_ONLY", "1"),
               ("stream_gathers_ms", "DPSO_SCAN_STREAM_ONLY", "2")))
    for name, var, val in probes:
        os.environ[var] = val
        try:
            p = dict(params, max_generations=gens + 4,
                     stall_generations=gens + 4)
            s = DiscreteSwarmSolver(**p)
            ctx = s._make_context(cost)
            try:
                if RNG == "numpy":
                    ctx.set_streams(numpy_stream_states(p["random_state"],
                                                        P + 2))
                ctx.init(seed_body, n_seed)
                ctx.step_timed(2)
                ms = []
                for _ in range(gens):
                    c0 = ctx.ctl()["two_opt_count"]
                    ph, cnt = ctx.step_timed(1)
                    if cnt > c0:
                        ms.append(float(ph[3]))
                if ms:
                    out[name] = float(np.median(ms))
            finally:
                ctx.close()
        finally:
            os.environ.pop(var, None)
    return out


def load_gather_peaks():
    try:
        with open(os.path.join(ROOT, "profiles", "r02",
                               "gather_peaks.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def load_gather4_peaks():
    try:
        with open(os.path.join(ROOT, "profiles", "r02",
                               "gather4_probe.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def gather4_stream_peak(peaks, line):
    """Measured L2 -> shared-memory row stream with TMA gather4 (four rows
    per copy), 32 rows per stage, 4 issuing warps (tools/gather4_probe.cu,
    profiles/r02/gather4_probe.json), scaled like row_stream_peak."""
    meas = {}
    for k, v in peaks.items():
        if k.startswith("gather4_") and k.endswith("B_w4"):
            size = int(k[len("gather4_"):].split("B")[0])
            meas[size] = float(v["tbs"]) * 1e3
    if not meas:
        return None, None
    near = min(meas, key=lambda z: abs(math.log(z / line)))
    cap = max(meas.values())
    return min(cap, meas[near] * line / near), near


def row_stream_peak(peaks, line):
    """Measured L2 -> shared-memory bulk-copy bandwidth (GB/s) for rows of
    `line` bytes, 32 rows per stage, 4 issuing warps (tools/gather_peaks.cu,
    profiles/r02/gather_peaks.json).  The rate is per copy at these sizes,
    so other row sizes scale from the nearest measured one, capped at the
    largest measured bandwidth."""
    meas = {}
    for k, v in peaks.items():
        if k.startswith("bulk_rows") and "_warps4_" in k:
            size = int(k[len("bulk_rows"):].split("_")[0])
            meas[size] = max(meas.get(size, 0.0), float(v["gbs"]))
    if not meas:
        return None, None
    near = min(meas, key=lambda z: abs(math.log(z / line)))
    cap = max(meas.values())
    return min(cap, meas[near] * line / near), near


def run_ours(args, cfg_name, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    from paper_1706_04399_b200.islands import IslandExchange
    from paper_1706_04399_b200.solver import numpy_stream_states

    cost, seed_tour = make_matrix(cfg)
    n, P = cost.shape[0], cfg["P"]
    W, K = args.warmup, args.steps
    G = W + K + args.profile_gens + 1
    # seed 7 on rank 0: the e2e run's and the reference trajectory's seed
    # (the per-generation cost depends on how often the 2-opt scan fires,
    # which the trajectory decides)
    params = gpu_params(cfg, P, G, 7 + rank)
    if seed_tour is not None:
        params["seed_tour"] = seed_tour
    solver = DiscreteSwarmSolver(**params)
    seed_body, n_seed = solver._seed(n)
    ctx = solver._make_context(cost)
    band = int(ctx.lib.dpso_scan_band(ctx.h))
    staging = int(ctx.lib.dpso_band_staging(ctx.h))
    band_line = int(ctx.lib.dpso_band_line(ctx.h))
    band_rows = int(ctx.lib.dpso_band_rows(ctx.h))
    bound = max(0, int(ctx.lib.dpso_scan_bound(ctx.h)))

    def bound_counters():
        pr = ctypes.c_ulonglong(0)
        ctx.lib.dpso_bound_pairs(ctx.h, ctypes.byref(pr))
        return int(ctx.lib.dpso_band_runs(ctx.h)), int(pr.value)
    if RNG == "numpy":
        ctx.set_streams(numpy_stream_states(params["random_state"], P + 2))
    ctx.init(seed_body, n_seed)
    ex = IslandExchange(ctx, n) if world > 1 else None

    ctx.step(W)
    torch.cuda.synchronize()
    scans0 = ctx.ctl()["two_opt_count"]
    runs0, _ = bound_counters()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(K):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
            ctx.step(1)
            if ex is not None and (k + 1) % args.exchange_every == 0:
                # island gbest exchange, inside the timed step; stream-
                # ordered (pack, NCCL all_gather, adopt): no host sync
                ex.exchange_device()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    scans_timed = ctx.ctl()["two_opt_count"] - scans0
    runs_timed = bound_counters()[0] - runs0  # passes with band-scan work
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = P * K * world / (total_ms / 1e3)

    # live per-phase kernel timing for the roofline (CUDA events on the
    # launching stream, same generations continued)
    c0 = ctx.ctl()
    runs_p0, pairs_p0 = bound_counters()
    prof_gens = args.profile_gens
    phase_ms, cnt = ctx.step_timed(prof_gens)
    fired = cnt - c0["two_opt_count"]
    runs_p1, pairs_p1 = bound_counters()
    names = ["update", "mutation", "select", "two_opt_scan", "two_opt_apply",
             "finalize"]
    phases = {k: v / prof_gens for k, v in zip(names, phase_ms)}
    ctx.close()

    # e2e through the public API with host buffers (H2D of the matrix and
    # RNG states, D2H of tour + convergence inside the timed region); with
    # N ranks: the island model's public API (IslandSolver, one island per
    # rank, gbest exchange every --exchange-every generations), timed
    # between barriers, max over ranks
    e2e, e2e_solver, e2e_params = None, None, None
    if not args.no_e2e:
        Ge = cfg["G"]
        ep = gpu_params(cfg, P, Ge, 7)
        if seed_tour is not None:
            ep["seed_tour"] = seed_tour
        # one short untimed fit first (module and pool warm-up, as the
        # timed steps have theirs)
        DiscreteSwarmSolver(**dict(ep, max_generations=max(1, W),
                                   stall_generations=max(1, W))).fit(cost)
        if world > 1:
            from paper_1706_04399_b200 import IslandSolver
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s = IslandSolver(exchange_every=args.exchange_every,
                             **ep).fit(cost)
            torch.cuda.synchronize()
            dt_t = torch.tensor([time.perf_counter() - t0],
                                dtype=torch.float64, device=dev)
            dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
            dt = float(dt_t.item())
            api = (f"IslandSolver(exchange_every={args.exchange_every})"
                   f".fit(host numpy matrix), {world} ranks")
        else:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s = DiscreteSwarmSolver(**ep).fit(cost)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            api = "DiscreteSwarmSolver.fit(host numpy matrix)"
        gens = s.n_generations_
        h2d = cost.nbytes + (P + 2) * 48 + (2 * n if seed_tour else 0)
        d2h = 4 * (n + 1) + 8 * (gens + 1)
        e2e = {"value": P * world * gens / dt, "unit": UNIT,
                       "h2d_bytes_per_step": h2d * world / gens,
                       "d2h_bytes_per_step": d2h * world / gens,
                       "generations": gens, "wall_s": dt, "api": api}
        e2e_solver, e2e_params = s, ep

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    gpk = load_gather_peaks()
    scan_alg = P * 4.0 * n * (n - 1)  # 8 B x n(n-1)/2 pairs
    upd_bytes = P * 26.0 * n           # update 16n + fitness 10n
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
    except Exception:
        tr = {}
    def update_roof():
        dur = phase_ms[0] / prof_gens
        alg = upd_bytes
        achieved = alg / (dur / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "update", "achieved": achieved,
                "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": tr.get(f"{cfg_name}:update"),
                "algorithmic_bytes_per_launch": alg,
                "avg_launch_ms": dur,
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)"}
        wf = tr.get(f"{cfg_name}:update:smem_wavefronts")
        if wf:
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            pk = sms * 1.965e9
            roof["binding"] = {
                "resource": "shared-memory pipe (wavefronts)",
                "wavefronts_per_launch": wf,
                "achieved_per_s": wf / (dur / 1e3), "peak_per_s": pk,
                "frac": wf / (dur / 1e3) / pk,
                "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared."
                          "sum per launch (profiles/ncu_traffic.json); peak "
                          f"= {sms} SMs x 1 wavefront/clock x 1.965 GHz"}
        return roof

    if cfg.get("ee", True) and fired > 0 and bound:
        # the bounded scan (k_two_opt_bound.cu): per particle it reads the
        # tour (2 B/row), d (8 B/row) and the two end points' row/column
        # minima (2 x 16 B/row, an L1-resident table), then gathers two fp64
        # entries per evaluated pair from the L2-resident matrix; random
        # 8-B gathers from L2 are its binding resource
        dom, dur_ms = "two_opt_scan", phase_ms[3] / fired
        traffic = tr.get(f"{cfg_name}:two_opt_bound")
        pairs = (pairs_p1 - pairs_p0) / fired
        # two kinds of bytes, two roofs: the tour and d rows stream
        # (coalesced, 10 B/row) at the measured sequential L2 read rate;
        # the evaluated pairs gather 2 x 8 B at random at the measured
        # random fp64 L2 gather rate.  (The city minima, an L1-resident
        # 8 B/city table, are left out: a lower floor, a lower fraction.)
        # frac = the sum of the two floors over the launch time
        seq_b = float(P) * n * (2 + 8)
        gat_b = 16.0 * pairs
        seq_pk = gpk.get("l2_seq_read_32MB", {}).get("gbs", 8993.4)
        gat_pk = gpk.get("gather_f64_8MB", {}).get("useful_gbs", 2288.7)
        floor_ms = (seq_b / seq_pk + gat_b / gat_pk) / 1e6
        alg = seq_b + gat_b
        achieved = alg / (dur_ms / 1e3) / 1e9
        peak = alg / (floor_ms / 1e3) / 1e9
        roof = {"bound": "l2", "kernel": "two_opt_scan (bounded)",
                "scan": "bounded (exact pair bound) + band fallback",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": floor_ms / dur_ms,
                "traffic": traffic,
                "algorithmic_bytes_per_launch": alg,
                "stream_bytes_per_launch": seq_b,
                "gather_bytes_per_launch": gat_b,
                "floor_ms": floor_ms,
                "pairs_evaluated_per_launch": pairs,
                "pairs_total_per_launch": P * n * (n - 1) / 2.0,
                "pair_fraction": pairs / (P * n * (n - 1) / 2.0),
                "band_fallback_passes": f"{runs_p1 - runs_p0}/{fired}",
                "band_fallback_passes_timed": f"{runs_timed}/{scans_timed}",
                "full_scan_equivalent_fp64_gbs":
                    scan_alg / (dur_ms / 1e3) / 1e9,
                "avg_launch_ms": dur_ms,
                "peak_source": "measured (profiles/r02/gather_peaks.json, "
                               "tools/gather_peaks.cu): sequential L2 reads "
                               f"{seq_pk:.0f} GB/s for the tour and d rows, "
                               f"random fp64 L2 gathers {gat_pk:.0f} GB/s "
                               "for the evaluated pairs; peak = the "
                               "combined rate of that byte mix",
                "note": "exact pruning: delta(i,j) >= -(h_i + h_j) skips "
                        "every pair that cannot reach the best delta found "
                        "so far; the rest are evaluated in fp64 (the "
                        "reference's argmin bit for bit).  The kernel is "
                        "latency-bound (a chain of dependent phases per "
                        "particle), far from both byte roofs.  The scan "
                        "phase includes the band scan launch for the "
                        "particles it hands over (empty in most passes)"}
    elif cfg.get("ee", True) and fired > 0:
        dom, dur_ms = "two_opt_scan", phase_ms[3] / fired
        traffic = tr.get(f"{cfg_name}:{dom}")
        # the binding resource of the scan: the cost rows it stages from L2
        # into shared memory.  Band scan: every row of the particle's tour
        # once, as int16 lines of round_up(2n + 12, 16) B (33 bands of 32
        # rows at n = 1000: the 31-row bands overlap by one row).  Column
        # scan: fp16/fp32 rows once per task.
        if band:
            # int16 rows (int8 past n ~ 1400), 32-slot bands of 31 pair
            # rows or 64-slot bands of 63 (two rows per lane): either way
            # every row of the tour is staged once per band it falls in
            line_b = band_line
            nbands = (n + band_rows - 2) // band_rows
            staged = float(P) * nbands * min(band_rows + 1, n) * line_b
        else:
            line_b = int(math.ceil(2 * n / 16.0) * 16)
            staged = float(P) * (n + 1) * line_b * max(1, -(-n // 1024))
        achieved = staged / (dur_ms / 1e3) / 1e9
        if staging == 2:
            peak, near = gather4_stream_peak(load_gather4_peaks(), line_b)
            peak_desc = (f"measured: L2->shared TMA gather4 row stream, "
                         f"{near}-B rows, 32 per stage, 4 issuing warps "
                         f"(profiles/r02/gather4_probe.json, "
                         f"tools/gather4_probe.cu), scaled to {line_b}-B "
                         f"rows")
        else:
            peak, near = row_stream_peak(gpk, line_b)
            peak_desc = (f"measured: L2->shared bulk-copy row stream, "
                         f"{near}-B rows, 32 per stage, 4 issuing "
                         f"warps (profiles/r02/gather_peaks.json, "
                         f"tools/gather_peaks.cu), scaled to "
                         f"{line_b}-B rows")
        roof = {"bound": "l2", "kernel": dom,
                "scan": ("band-exact", "band-filter")[band - 1]
                if band else "column",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if peak else None,
                "traffic": traffic,
                "staged_bytes_per_launch": staged,
                "algorithmic_fp64_bytes_per_launch": scan_alg,
                "algorithmic_fp64_gbs": scan_alg / (dur_ms / 1e3) / 1e9,
                "avg_launch_ms": dur_ms,
                "staging": {0: "column scan", 1: "bulk copies",
                            2: "TMA gather4"}.get(staging),
                "row_line_bytes": line_b,
                "pair_rows_per_band": band_rows if band else None,
                "peak_source": peak_desc,
                "l2_random_gather_f64_gbs":
                    gpk.get("gather_f64_8MB", {}).get("useful_gbs"),
                "note": "the matrix is L2-resident and each staged row "
                        "serves a whole band of pairs, so the kernel is "
                        "bound by the L2->SMEM row stream and SM issue, "
                        "not by HBM"}
    else:
        dom, dur_ms = "update", phase_ms[0] / prof_gens
        roof = update_roof()
        traffic = roof["traffic"]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": total_ms / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg_name, cfg, args, world),
        "gpu_launches": gpu_launch_count(cfg, W + 1, K, band=band,
                                         bound=bound),
        "roofline": roof,
        "roofline_update": update_roof() if dom != "update" else None,
        "phase_ms_per_gen": phases,
        "two_opt_fired": f"{fired}/{prof_gens}",
        "two_opt_scans_timed": f"{scans_timed}/{K}",
    }
    # the scan's own floor, live (the same launch reduced to its row stream)
    if cfg.get("ee", True) and world == 1 and dom == "two_opt_scan" \
            and not bound:
        try:
            fl = scan_floors(cost, params, seed_body, n_seed, P, band=band)
            if fl.get("stream_only_ms"):
                fl["frac_of_stream_only"] = fl["stream_only_ms"] / dur_ms
            if fl:
                line["roofline"]["floors"] = fl
        except Exception as exc:  # a probe failing must not lose the line
            line["roofline"]["floors"] = {"error": str(exc)[:200]}
    # clocks
    line["clocks"] = clk.summary()
    if e2e is not None:
        line["e2e"] = e2e

    if not args.no_e2e:
        s, ep = e2e_solver, e2e_params
        # time-to-reference-best tour length (BASELINE metric, second part):
        # with numpy-exact streams this run IS the reference's run for this
        # seed (bit for bit), so the reference's best over the schedule is
        # conv[-1] and it is first reached at generation g*; a fit capped at
        # g* generations times how long this path takes to reach it
        if RNG == "numpy" and world == 1:
            conv = list(s.convergence_)
            g_star = next(i for i, c in enumerate(conv) if c == conv[-1])
            g_run = max(1, g_star)
            tp = dict(ep, max_generations=g_run, stall_generations=g_run)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            s2 = DiscreteSwarmSolver(**tp).fit(cost)
            torch.cuda.synchronize()
            t_best = time.perf_counter() - t1
            assert s2.best_fitness_ == conv[-1]
            line["time_to_reference_best"] = {
                "value": t_best, "unit": "s", "higher_is_better": False,
                "reference_best": conv[-1], "generation": g_star,
                "schedule": gens,
                "note": "fit() wall time (host matrix in, tour out) to the "
                        "reference's best tour length over the schedule for "
                        "this seed; numpy-exact streams make this the "
                        "reference's own trajectory"}
            # the unmodified reference's own run of this instance and seed
            # (tests/golden/make_golden_c2.py, one core of the build host)
            gp = os.path.join(ROOT, "tests", "golden", "golden_c2_full.json")
            if cfg_name == "c2" and os.path.exists(gp):
                with open(gp) as fh:
                    g = json.load(fh)
                pr = g["params"]
                if (pr["random_state"] == ep["random_state"]
                        and pr["n_particles"] == P
                        and pr["max_generations"] == Ge):
                    line["time_to_reference_best"]["reference_run"] = {
                        "reference_best": g["best_fitness"],
                        "trajectory_identical": conv == g["convergence"],
                        "reference_time_to_best_s":
                            g["reference_time_to_best_s"],
                        "reference_generation": g["best_generation"],
                        "reference_wall_s": g["reference_wall_s"],
                        "host": g["host"],
                        "fixture": "tests/golden/golden_c2_full.json"}

    if not args.no_cpu_baseline and world == 1:
        rate, g, dt = cpu_sample(cost, cfg, seed_tour=seed_tour)
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"oracle port (oracle/dpso_oracle.py) of the reference"
                       f" solve, 32-particle swarm on the same matrix, 1 warm"
                       f"-up + {g} timed generations ({dt:.1f}s), 1 thread")}
        ttb = line.get("time_to_reference_best")
        if ttb is not None and "reference_run" not in ttb:
            # no measured reference run for this config: the reference
            # (single-threaded, parallel=False) needs g* generations of P
            # particles at the port's one-core rate
            ttb["reference_cpu_estimate_s"] = ttb["generation"] * P / rate
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--exchange-every", type=int, default=10)
    ap.add_argument("--profile-gens", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rng", choices=["numpy", "philox"], default=None,
                    help="numpy: the reference's PCG64 streams bit for bit; "
                         "philox: counter-based production RNG (default: "
                         "the config's; numpy except C5)")
    ap.add_argument("--scan-mode", choices=["auto", "fp64", "exact32",
                                            "filter32"], default="auto",
                    help="force the 2-opt scan mode (default: chosen from "
                         "the matrix)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    global RNG
    RNG = args.rng or cfg.get("rng", "numpy")
    if args.scan_mode != "auto":
        os.environ["DPSO_SCAN_MODE"] = {"fp64": "0", "exact32": "1",
                                        "filter32": "2"}[args.scan_mode]
    if args.impl == "reference":
        run_reference(args, args.config, cfg)
        return
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        sys.exit(launch_ranks(args))
    if world and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: "
                 f"one rank per GPU is required")
    run_ours(args, args.config, cfg)


def launch_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: start N ranks (one per
    GPU) with torch.distributed.run on this node and wait for them; fail
    loudly when the node has fewer than N GPUs."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} "
                         f"GPUs, this node has {have}\n")
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
