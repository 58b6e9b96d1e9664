"""ncu driver at the C3 shape (N=500 grid costs: EXACT32 on fp16 rows,
P=16384): a few generations of the swarm (update, mutation, 2-opt)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import math  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def main():
    n, P = 500, 16384
    side = int(math.ceil(math.sqrt(n)))
    idx = np.arange(n)
    pts = np.stack([idx % side, idx // side], 1).astype(float)
    cost = np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)
    s = DiscreteSwarmSolver(n_particles=P, max_generations=10,
                            stall_generations=10, random_state=1)
    ctx = s._make_context(cost)
    ctx.set_streams(numpy_stream_states(1, P + 2))
    ctx.init(None, 0)
    ctx.step(int(os.environ.get("PROF_GENS", "3")))
    torch.cuda.synchronize()
    print("ok", ctx.ctl())
    ctx.close()


if __name__ == "__main__":
    main()
