"""Small, deterministic driver for ncu captures of the hot kernels at the
C2 shape (N=1000, P=1024): a full-work 2-opt scan batch (random tours, so
every launch scans all pairs), then a few swarm generations (update,
mutation pipeline, select, 2-opt, finalize)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver, best_exchange_batch  # noqa
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def main():
    n = int(os.environ.get("PROF_N", "1000"))
    P = int(os.environ.get("PROF_P", "1024"))
    gens = int(os.environ.get("PROF_GENS", "4"))
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10.0
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    tours = np.stack([rng.permutation(n) for _ in range(P)]).astype(np.int32)
    for _ in range(2):
        best_exchange_batch(cost, tours)
    s = DiscreteSwarmSolver(n_particles=P, max_generations=100,
                            stall_generations=100, random_state=1)
    ctx = s._make_context(cost)
    ctx.set_streams(numpy_stream_states(1, P + 2))
    ctx.init(None, 0)
    ctx.step(gens)
    torch.cuda.synchronize()
    print("ok", ctx.ctl())
    ctx.close()


if __name__ == "__main__":
    main()
