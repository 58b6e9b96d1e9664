"""Per-generation update time for inertia w < 1 (the transposition-list
path, k_update_seq) against w = 1 (k_update_w1), C2 shape."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def main():
    n, P = 1000, 1024
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10.0
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    for w in (1.0, 0.9, 0.99):
        s = DiscreteSwarmSolver(n_particles=P, inertia=w, max_generations=400,
                                stall_generations=400, random_state=3)
        ctx = s._make_context(cost)
        ctx.set_streams(numpy_stream_states(3, P + 2))
        ctx.init(None, 0)
        out = []
        for block in range(4):
            ctx.step(40)
            ph, _ = ctx.step_timed(5)
            out.append(round(float(ph[0]) / 5, 3))
        ctx.close()
        print("w", w, "update ms/gen after 45/90/135/180 gens:", out)


if __name__ == "__main__":
    main()
