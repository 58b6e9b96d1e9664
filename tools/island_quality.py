"""Statistical quality of the island model ("end-to-end
best-tour length over 20 seeds statistically no worse than the reference").

For each seed: the reference's solve (numpy-exact streams: bit-identical to
the reference's own run) with P particles, against K islands of P
particles each whose gbest is exchanged every E generations (the winner:
smallest fitness, lowest island on ties; adopted iff strictly better - the
same rule as islands.py / dpso_island_adopt).  The islands run one after
the other on one GPU: this measures solution quality, not speed.
Usage: python tools/island_quality.py [n] [P] [G] [K] [E] [seeds]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    n, P, G, K, E, S = (a + [200, 128, 200, 4, 10, 20][len(a):])[:6]
    rng = np.random.default_rng(2024)
    pts = rng.random((n, 2)) * 10
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    ref, isl = [], []
    for seed in range(S):
        params = dict(n_particles=P, max_generations=G, stall_generations=G,
                      random_state=seed)
        ref.append(DiscreteSwarmSolver(**params).fit(cost).best_fitness_)
        ctxs = []
        for k in range(K):
            p = dict(params, random_state=seed * 1000 + k)
            s = DiscreteSwarmSolver(**p)
            ctx = s._make_context(cost)
            ctx.set_streams(numpy_stream_states(p["random_state"], P + 2))
            ctx.init(None, 0)
            ctxs.append(ctx)
        done = 0
        while done < G:
            step = min(E, G - done)
            for ctx in ctxs:
                ctx.step(step)
            done += step
            res = [ctx.result() for ctx in ctxs]
            fits = [(r[1], k) for k, r in enumerate(res)]
            wfit, wk = min(fits)
            for k, ctx in enumerate(ctxs):
                if k != wk and wfit < res[k][1]:
                    ctx.offer_gbest(np.asarray(res[wk][0][:n]), wfit)
        isl.append(min(ctx.result()[1] for ctx in ctxs))
        for ctx in ctxs:
            ctx.close()
    ref, isl = np.array(ref), np.array(isl)
    out = {"n": n, "P_per_island": P, "generations": G, "islands": K,
           "exchange_every": E, "seeds": S,
           "reference_mean": float(ref.mean()),
           "islands_mean": float(isl.mean()),
           "reference_median": float(np.median(ref)),
           "islands_median": float(np.median(isl)),
           "islands_no_worse_seeds": int((isl <= ref).sum())}
    try:
        from scipy.stats import wilcoxon
        out["wilcoxon_p_islands_worse"] = float(
            wilcoxon(isl, ref, alternative="greater").pvalue)
    except Exception as exc:  # noqa: BLE001
        out["wilcoxon"] = str(exc)[:120]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
