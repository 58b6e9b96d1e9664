"""Per-phase device time across a whole solve, in blocks of generations
(dpso_step_timed), to see how the cost of a generation drifts as the swarm
converges.  Env: GP_N, GP_P, GP_G, GP_BLOCK."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402

PH = ("update", "mutation", "select", "scan", "apply", "finalize")


def main():
    n = int(os.environ.get("GP_N", "1000"))
    P = int(os.environ.get("GP_P", "1024"))
    G = int(os.environ.get("GP_G", "500"))
    B = int(os.environ.get("GP_BLOCK", "50"))
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10.0
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    s = DiscreteSwarmSolver(n_particles=P, max_generations=G,
                            stall_generations=G, random_state=7)
    ctx = s._make_context(cost)
    ctx.set_streams(numpy_stream_states(7, P + 2))
    ctx.init(None, 0)
    done = 0
    last = 0
    while done < G:
        b = min(B, G - done)
        ms, cnt = ctx.step_timed(b)
        done += b
        print(f"gens {done - b + 1:4d}-{done:4d} 2opt {cnt - last:3d}/{b} "
              + " ".join(f"{k} {v / b:.3f}" for k, v in zip(PH, ms))
              + f" total {ms.sum() / b:.3f} ms/gen", flush=True)
        last = cnt
    ctx.close()


if __name__ == "__main__":
    main()
