"""How often the 2-opt scan fires over a C2 solve (500 generations), by
seed: the scan runs for all particles only in generations where the update
and mutation did not strictly improve gbest (solver.py:307-319), so the
per-generation cost of a solve depends on its trajectory.

    python tools/scan_fraction.py > profiles/r02/scan_fraction_c2.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    cfg = bench.CONFIGS["c2"]
    cost, _ = bench.make_matrix(cfg)
    rows = []
    for seed in (0, 1, 2, 3, 7, 11, 42, 1000, 1001, 2024):
        s = DiscreteSwarmSolver(**bench.gpu_params(cfg, cfg["P"], cfg["G"],
                                                   seed))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.fit(cost)
        dt = time.perf_counter() - t0
        conv = s.convergence_
        improved = sum(1 for a, b in zip(conv, conv[1:]) if b < a)
        rows.append({"seed": seed, "generations": s.n_generations_,
                     "gbest_improved_gens": improved,
                     "fit_s": round(dt, 4),
                     "e2e_particle_iter_per_s": round(
                         cfg["P"] * s.n_generations_ / dt),
                     "best": s.best_fitness_})
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"config": "c2", "runs": rows}))


if __name__ == "__main__":
    main()
