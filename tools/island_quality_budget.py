"""Equal-budget solution quality of the island model (SURVEY §8(e):
"end-to-end best-tour length over 20 seeds statistically no worse than the
reference").

Per seed: the reference's solve with P particles (numpy-exact streams: the
reference's own run, bit for bit) against the public island API
(``IslandSolver``) with K islands of P/K particles each - the same number
of particle-iterations per generation - exchanging gbest every E
generations, the same generation schedule.  The islands run as the local
mode's threads on one GPU: this measures quality, not speed.  Reports both
means, the seeds where the islands are no worse, and one-sided Wilcoxon
signed-rank p-values in both directions.

Usage: python tools/island_quality_budget.py [n] [P] [G] [K] [E] [seeds]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver, IslandSolver  # noqa


def main():
    a = [int(x) for x in sys.argv[1:]]
    n, P, G, K, E, S = (a + [200, 128, 200, 4, 10, 20][len(a):])[:6]
    rng = np.random.default_rng(2024)
    pts = rng.random((n, 2)) * 10
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    ref, isl = [], []
    for seed in range(S):
        params = dict(max_generations=G, stall_generations=G,
                      random_state=seed)
        ref.append(DiscreteSwarmSolver(n_particles=P, **params)
                   .fit(cost).best_fitness_)
        s = IslandSolver(exchange_every=E, devices=["cuda:0"] * K,
                         n_particles=P // K, **params).fit(cost)
        isl.append(s.best_fitness_)
    ref, isl = np.array(ref), np.array(isl)
    out = {"n": n, "P_reference": P, "islands": K, "P_per_island": P // K,
           "generations": G, "exchange_every": E, "seeds": S,
           "budget": "equal: K x P/K particle-iterations per generation",
           "reference_mean": float(ref.mean()),
           "islands_mean": float(isl.mean()),
           "reference_median": float(np.median(ref)),
           "islands_median": float(np.median(isl)),
           "islands_no_worse_seeds": int((isl <= ref).sum()),
           "reference": ref.tolist(), "islands_best": isl.tolist()}
    from scipy.stats import wilcoxon
    out["wilcoxon_p_islands_worse"] = float(
        wilcoxon(isl, ref, alternative="greater").pvalue)
    out["wilcoxon_p_islands_better"] = float(
        wilcoxon(isl, ref, alternative="less").pvalue)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
