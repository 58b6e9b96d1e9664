"""Statistical parity of the Philox production RNG (rng="philox") against
the numpy-exact streams (the reference's own runs) at bench-like sizes
(round-1 verdict: the only Philox quality check was one 36-node scene).

Per seed s: DiscreteSwarmSolver(random_state=s) in both RNG modes on the
same random-Euclidean instance; reports the mean / median best tour
lengths and a two-sided Wilcoxon signed-rank p-value (H0: the two modes
give the same distribution of best tours), plus one-sided p-values.

Usage: python tools/philox_quality.py [n] [P] [G] [seeds]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    n, P, G, S = (a + [1000, 256, 100, 20][len(a):])[:4]
    rng = np.random.default_rng(77)
    pts = rng.random((n, 2)) * 10
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    res = {"numpy": [], "philox": []}
    for seed in range(S):
        for mode in res:
            s = DiscreteSwarmSolver(n_particles=P, max_generations=G,
                                    stall_generations=G, random_state=seed,
                                    rng=mode).fit(cost)
            res[mode].append(s.best_fitness_)
    a_np, a_ph = np.array(res["numpy"]), np.array(res["philox"])
    from scipy.stats import wilcoxon
    out = {"n": n, "P": P, "generations": G, "seeds": S,
           "numpy_mean": float(a_np.mean()), "philox_mean": float(a_ph.mean()),
           "numpy_median": float(np.median(a_np)),
           "philox_median": float(np.median(a_ph)),
           "relative_mean_diff": float((a_ph.mean() - a_np.mean()) /
                                       a_np.mean()),
           "wilcoxon_p_two_sided": float(wilcoxon(a_ph, a_np).pvalue),
           "wilcoxon_p_philox_worse": float(
               wilcoxon(a_ph, a_np, alternative="greater").pvalue),
           "numpy": a_np.tolist(), "philox": a_ph.tolist()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
