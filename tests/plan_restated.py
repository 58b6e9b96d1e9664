"""Test infrastructure: the reference CLI's ``plan`` outputs restated
around this package's drop-in ``build_graph`` and ``DiscreteSwarmSolver``.

Follows pipeline.py:33-61 (plan_inspection: build_graph -> solver.fit on
graph.cost with the boustrophedon seed -> validate_tour / tour_length
check) and cli.py:122-173 (_tour_document, the three output files), with
the reference's CoveragePlan / VoxelGrid replaced by the recorded inputs of
tests/golden/golden_plan.json.  Only tests import this module."""
import argparse
import json
import os

import numpy as np


class Grid:
    """voxel.py:46-66 (the members build_graph and the CLI use)."""

    def __init__(self, rec):
        self.dims = tuple(rec["dims"])
        self.origin = np.asarray(rec["origin"], dtype=float)
        self.voxel_size = float(rec["voxel_size"])
        n = int(np.prod(self.dims))
        bits = np.unpackbits(np.asarray(rec["occ"], dtype=np.uint8))[:n]
        self.occupancy = bits.astype(bool).reshape(self.dims)

    def center(self, idx):
        return self.origin + (np.asarray(idx, dtype=float) + 0.5) * \
            self.voxel_size

    def point_to_voxel(self, point):
        rel = (np.asarray(point, dtype=float) - self.origin) / self.voxel_size
        idx = np.clip(np.floor(rel).astype(int), 0,
                      np.asarray(self.dims) - 1)
        return (int(idx[0]), int(idx[1]), int(idx[2]))

    def is_free(self, idx):
        return not bool(self.occupancy[idx])


class Viewpoint:
    def __init__(self, rec):
        self.id = rec["id"]
        self.position = np.asarray(rec["position"], dtype=float)
        self.orientation = np.asarray(rec["orientation"], dtype=float)
        self.surface_index = rec["surface_index"]


class Plan:
    def __init__(self, recs):
        self.viewpoints = [Viewpoint(r) for r in recs]


def solver_params(argv):
    """cli.py:43-70 defaults and flags."""
    p = argparse.ArgumentParser()
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--particles", type=int, default=100)
    p.add_argument("--generations", type=int, default=200)
    p.add_argument("--stall", type=int, default=30)
    p.add_argument("--mutation-period", type=int, default=3)
    p.add_argument("--seed-fraction", type=float, default=0.1)
    p.add_argument("--heuristic", default="admissible")
    a = p.parse_args(argv)
    return dict(n_particles=a.particles, max_generations=a.generations,
                stall_generations=a.stall, mutation_period=a.mutation_period,
                seed_fraction=a.seed_fraction, use_mutation=True,
                use_edge_exchange=True, parallel=False, random_state=a.seed)


def run_plan(pkg, rec, out_dir):
    """Writes tour.json, convergence.csv, cost_matrix.txt into out_dir and
    returns their contents."""
    grid = Grid(rec["grid"])
    plan = Plan(rec["viewpoints"])
    graph = pkg.build_graph(plan, grid, tuple(rec["weights"]),
                            heuristic_mode=rec["heuristic"])
    params = solver_params(rec["argv"])
    solver = pkg.DiscreteSwarmSolver(seed_tour=tuple(rec["seed_tour"]),
                                     **params)
    solver.fit(graph.cost)
    tour = solver.best_tour_
    body = list(tour[:-1])
    assert tour[0] == tour[-1] and sorted(body) == list(range(graph.n_nodes))
    seq = np.asarray(tour, dtype=int)
    assert abs(float(graph.cost[seq[:-1], seq[1:]].sum()) -
               solver.best_fitness_) < 1e-9
    report = solver.report_
    legs = []
    for a, b in zip(tour[:-1], tour[1:]):
        leg = graph.leg(a, b)
        legs.append({
            "from": int(a), "to": int(b),
            "cost": float(graph.cost[a, b]),
            "virtual": bool(graph.virtual[a, b]),
            "waypoints": ([[float(c) for c in grid.center(w)]
                           for w in leg.waypoints] if leg else []),
        })
    doc = {
        "total_cost": report.best_fitness,
        "generations": report.generations_run,
        "viewpoint_order": [int(x) for x in tour],
        "viewpoints": [
            {"id": vp.id, "position": [float(c) for c in vp.position],
             "orientation": [float(c) for c in vp.orientation],
             "surface_index": vp.surface_index}
            for vp in plan.viewpoints],
        "legs": legs,
    }
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "tour.json"), "w") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")
    with open(os.path.join(out_dir, "convergence.csv"), "w") as fh:
        fh.write("generation,best_fitness\n")
        for g, fit in enumerate(report.convergence):
            fh.write(f"{g},{fit!r}\n")
    pkg.save_cost_matrix(os.path.join(out_dir, "cost_matrix.txt"), graph.cost)
    return {f: open(os.path.join(out_dir, f)).read()
            for f in ("tour.json", "convergence.csv", "cost_matrix.txt")}
