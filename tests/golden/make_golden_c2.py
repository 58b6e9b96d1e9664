"""Golden trajectories of the UNMODIFIED reference at the bench's headline
instance (BASELINE configs[1], bench.py ``--config c2``).

Run in the build container only (``/root/reference`` does not exist on the GPU
box)::

    python tests/golden/make_golden_c2.py --gens 8 --seed 1000 --out golden_c2_g8.json
    python tests/golden/make_golden_c2.py --gens 500 --seed 7 --out golden_c2_full.json

Instance: ``random_euclidean_matrix(1000, default_rng(1000))``
(conftest.py:27-31; bench.py ``make_matrix``), ``DiscreteSwarmSolver(
n_particles=1024, max_generations=G, stall_generations=G,
random_state=seed)`` with the paper defaults (solver.py:118-135), i.e. the
exact call bench.py's e2e leg makes (seed 7, G=500) and its timed swarm
(seed 1000).

The reference's ``fit`` is called unmodified.  The only addition is a
subclass whose ``_update_particle`` notes the wall time at which each
generation's first particle update starts (it then calls the reference's
own method), so the fixture also records the reference's own time to reach
its best tour length on this host (one core, ``parallel=False``).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import resource
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from conftest import random_euclidean_matrix  # noqa: E402
from inspectour.solver import DiscreteSwarmSolver  # noqa: E402


class _Timed(DiscreteSwarmSolver):
    """Records the perf_counter time of each generation's first update."""

    def _update_particle(self, p, gbest_body, cost_rows):
        if self._calls % self.n_particles == 0:
            self._gen_t.append(time.perf_counter())
        self._calls += 1
        return super()._update_particle(p, gbest_body, cost_rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1000)
    ap.add_argument("--particles", type=int, default=1024)
    ap.add_argument("--out", default="golden_c2_g8.json")
    args = ap.parse_args()

    cost = random_euclidean_matrix(1000, np.random.default_rng(1000))
    G = args.gens
    s = _Timed(n_particles=args.particles, max_generations=G,
               stall_generations=G, random_state=args.seed)
    s._calls, s._gen_t = 0, []
    t0 = time.perf_counter()
    s.fit(cost)
    wall = time.perf_counter() - t0
    conv = list(s.convergence_)
    g_star = next(i for i, c in enumerate(conv) if c == conv[-1])
    # generation g's update starts at _gen_t[g-1]; its best is known at the
    # start of generation g+1 (or at the end of the fit)
    ends = s._gen_t[1:] + [t0 + wall]
    t_best = (ends[g_star - 1] - t0) if g_star > 0 else 0.0
    out = {
        "instance": "random_euclidean_matrix(1000, default_rng(1000))",
        "params": {"n_particles": args.particles, "max_generations": G,
                   "stall_generations": G, "random_state": args.seed},
        "best_tour": list(s.best_tour_),
        "best_fitness": s.best_fitness_,
        "convergence": conv,
        "n_generations": s.n_generations_,
        "reference_wall_s": wall,
        "reference_time_to_best_s": t_best,
        "best_generation": g_star,
        "host": {"cpu": platform.processor() or platform.machine(),
                 "threads": 1,
                 "max_rss_mb": resource.getrusage(
                     resource.RUSAGE_SELF).ru_maxrss / 1024.0},
    }
    with open(os.path.join(HERE, args.out), "w") as fh:
        json.dump(out, fh)
    print(json.dumps({k: v for k, v in out.items()
                      if k not in ("best_tour", "convergence")}))


if __name__ == "__main__":
    main()
