"""The algorithm-comparison harness of ``inspectour bench`` (cli.py:178-274)
on the device: every (instance, algorithm, trial) is an independent swarm,
and ``workers`` of them run concurrently, each on its own CUDA stream (one
host thread per stream; the C ABI releases the GIL while it waits).

Same algorithms and parameter overrides as cli.py:181-203 (``enhanced``,
``no_init``, ``no_mutation``, ``no_edge_exchange``, ``plain``, ``nn_2opt``),
same seeds (``seed + trial``), same ``results.csv`` / ``summary.csv`` files
(cli.py:240-272).  With the numpy-exact RNG every cost is the reference's,
bit for bit; only the wall times differ.
"""
from __future__ import annotations

import csv
import statistics
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .kernels import nearest_neighbor_two_opt
from .solver import DiscreteSwarmSolver, _torch

ALGORITHMS = ("enhanced", "no_init", "no_mutation", "no_edge_exchange",
              "plain", "nn_2opt")


@dataclass
class BenchResult:
    """baselines.BenchResult: one (algorithm, instance, seed) run."""
    algorithm: str
    instance: str
    seed: int
    cost: float
    wall_time: float
    effort: int


def solver_params(particles=100, generations=200, stall=30,
                  mutation_period=3, seed_fraction=0.1, no_init_seed=False,
                  no_mutation=False, no_edge_exchange=False, parallel=False,
                  seed=0) -> dict:
    """cli.py:60-71 with the CLI defaults (cli.py:44-56)."""
    return dict(n_particles=particles, max_generations=generations,
                stall_generations=stall, mutation_period=mutation_period,
                seed_fraction=0.0 if no_init_seed else seed_fraction,
                use_mutation=not no_mutation,
                use_edge_exchange=not no_edge_exchange, parallel=parallel,
                random_state=seed)


def _overrides(algo: str, seed_tour):
    """cli.py:191-203."""
    if algo == "enhanced":
        return dict(seed_tour=seed_tour)
    if algo == "no_init":
        return dict(seed_tour=None, seed_fraction=0.0)
    if algo == "no_mutation":
        return dict(seed_tour=seed_tour, use_mutation=False)
    if algo == "no_edge_exchange":
        return dict(seed_tour=seed_tour, use_edge_exchange=False)
    if algo == "plain":
        return dict(seed_tour=None, seed_fraction=0.0, use_mutation=False,
                    use_edge_exchange=False)
    raise ValueError(f"unknown algorithm {algo!r}")


def run_bench(instances, trials: int = 15, seed: int = 0, base=None,
              algorithms=ALGORITHMS, workers: int = 8, device=None,
              rng: str = "numpy"):
    """instances: [(name, cost (n x n), seed_tour or None)].  Returns the
    BenchResult rows in the reference's order (instance, algorithm, trial).
    """
    torch = _torch()
    base = dict(base or solver_params(seed=seed))
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    jobs = []
    for name, cost, seed_tour in instances:
        cost = np.asarray(cost, dtype=float)
        for algo in algorithms:
            for trial in range(trials):
                jobs.append((str(name), cost, seed_tour, algo, seed + trial))
    local = threading.local()

    def run(job):
        name, cost, seed_tour, algo, s = job
        if not hasattr(local, "stream"):
            torch.cuda.set_device(dev)
            local.stream = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(local.stream):
            t0 = time.perf_counter()
            if algo == "nn_2opt":  # cli.py:187-189
                _, value = nearest_neighbor_two_opt(cost)
                effort = 0
            else:
                params = dict(base)
                params.update(random_state=s, **_overrides(algo, seed_tour))
                solver = DiscreteSwarmSolver(**params, rng=rng, device=dev)
                solver.fit(cost)
                value = solver.report_.best_fitness
                effort = solver.report_.generations_run
            local.stream.synchronize()
            return BenchResult(algorithm=algo, instance=name, seed=s,
                               cost=float(value),
                               wall_time=time.perf_counter() - t0,
                               effort=int(effort))

    if workers <= 1:
        return [run(j) for j in jobs]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(run, jobs))


def write_results(out_dir, rows, instance_names) -> Path:
    """results.csv and summary.csv exactly as cli.py:240-272 writes them."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    results_path = out_dir / "results.csv"
    with open(results_path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["algorithm", "instance", "seed", "cost", "time",
                    "effort"])
        for r in rows:
            w.writerow([r.algorithm, r.instance, r.seed, repr(r.cost),
                        f"{r.wall_time:.6f}", r.effort])
    with open(out_dir / "summary.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["instance", "algorithm", "mean_cost", "sd_cost",
                    "mean_time", "improvement_vs_plain_pct"])
        for name in instance_names:
            by_algo = {}
            for r in rows:
                if r.instance == str(name):
                    by_algo.setdefault(r.algorithm, []).append(r)
            plain_mean = statistics.mean(
                x.cost for x in by_algo.get("plain", [])) if by_algo.get(
                    "plain") else None
            for algo, rs in by_algo.items():
                costs = [x.cost for x in rs]
                mean = statistics.mean(costs)
                sd = statistics.stdev(costs) if len(costs) > 1 else 0.0
                impr = ""
                if plain_mean:
                    impr = f"{100.0 * (plain_mean - mean) / plain_mean:.3f}"
                w.writerow([name, algo, f"{mean:.6f}", f"{sd:.6f}",
                            f"{statistics.mean(x.wall_time for x in rs):.6f}",
                            impr])
    return results_path
