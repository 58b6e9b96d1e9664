"""Wall time of the device bench harness (cli.py:178-274 defaults: 6
algorithms x 15 trials, P=100, G=200, stall 30) on the wall scene (N=15),
the ablation scene (N=36) and a random-Euclidean N=200 instance: serial
(workers=1) and concurrent (workers=W) on one GPU, against the oracle port
of the reference's CPU harness on one trial per (instance, algorithm),
scaled to 15 trials.  Usage: python tools/bench_harness_timing.py [W]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from conftest import random_euclidean_matrix  # noqa: E402
from oracle import dpso_oracle as O  # noqa: E402
from paper_1706_04399_b200.bench_harness import (ALGORITHMS, _overrides,  # noqa: E402
                                                run_bench, solver_params)


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    g = json.load(open(os.path.join(ROOT, "tests", "golden",
                                    "golden_e2e.json")))
    inst = [("wall", np.array(g["matrices"]["wall"], float),
             g["seed_tours"]["wall"]),
            ("ablation", np.array(g["matrices"]["ablation"], float),
             g["seed_tours"]["ablation"]),
            ("euclid200", random_euclidean_matrix(200,
                                                  np.random.default_rng(7)),
             None)]
    base = solver_params(seed=0)
    run_bench(inst[:1], trials=1, base=base, workers=2)  # warm-up
    out = {"runs": len(inst) * len(ALGORITHMS) * 15, "workers": W}
    for w in (1, W):
        t = time.perf_counter()
        rows = run_bench(inst, trials=15, base=base, workers=w)
        out[f"gpu_wall_s_workers{w}"] = time.perf_counter() - t
    # oracle port of the reference harness: one trial per pair, x15
    t = time.perf_counter()
    ref = {}
    for name, cost, st in inst:
        for algo in ALGORITHMS:
            if algo == "nn_2opt":
                ref[(name, algo)] = O.nearest_neighbor_two_opt(cost)[1]
                continue
            p = dict(base)
            p.update(random_state=0, **_overrides(algo, st))
            ref[(name, algo)] = O.OracleSolver(**p).fit(cost).best_fitness_
    out["cpu_port_one_trial_s"] = time.perf_counter() - t
    out["cpu_port_est_15_trials_s"] = 15 * out["cpu_port_one_trial_s"]
    out["seed0_costs_match"] = all(
        r.cost == ref[(r.instance, r.algorithm)] for r in rows if r.seed == 0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
