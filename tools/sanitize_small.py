"""Small end-to-end exercises of every kernel family for compute-sanitizer
(memcheck / racecheck): numpy-exact solve with 2-opt + mutation (fp16 and
fp32 rows, FILTER and EXACT), Philox solve, w < 1, batch 2-opt / NN, the
parallel init walk, and the cost-matrix build."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1706_04399_b200 as pkg  # noqa: E402


def euclid(n, seed):
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2)) * 10
    c = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(c, 0.0)
    return c


def main():
    c = euclid(150, 1)
    for kw in ({}, {"inertia": 0.5}, {"rng": "philox"},
               {"mutation_period": 1, "seed_fraction": 0.3,
                "seed_tour": list(range(150)) + [0]}):
        s = pkg.DiscreteSwarmSolver(n_particles=40, max_generations=6,
                                    stall_generations=6, random_state=2,
                                    **kw).fit(c)
        print(kw.get("rng", "numpy"), s.best_fitness_, s.n_generations_)
    ci = np.floor(c)
    s = pkg.DiscreteSwarmSolver(n_particles=40, max_generations=6,
                                stall_generations=6, random_state=3).fit(ci)
    print("int", s.best_fitness_)
    c2 = euclid(1100, 2)
    s = pkg.DiscreteSwarmSolver(n_particles=16, max_generations=3,
                                stall_generations=3, random_state=4).fit(c2)
    print("n1100", s.best_fitness_)
    tours = np.stack([np.random.default_rng(5).permutation(150)
                      for _ in range(8)]).astype(np.int32)
    pkg.best_exchange_batch(c, tours)
    pkg.tour_cost_batch(c, tours)
    print("nn2opt", pkg.nearest_neighbor_two_opt(c)[1])
    occ = np.zeros((12, 10, 6), bool)
    occ[4:6, 2:8, :4] = True
    vox = [(0, 0, 0), (11, 9, 5), (5, 0, 5), (2, 9, 1), (10, 1, 2)]
    cost, virt, vc = pkg.build_cost_matrix(occ, vox, (1.0, 1.0, 1.0))
    print("graph", cost.sum(), virt.sum(), vc)


if __name__ == "__main__":
    main()
