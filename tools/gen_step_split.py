"""Graph-mode step time of mutating vs plain generations (CUDA events around
each dpso_step(1)), to see what the mutation call costs on the critical
path.  Env: GS_N, GS_P, GS_G."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def main():
    n = int(os.environ.get("GS_N", "1000"))
    P = int(os.environ.get("GS_P", "1024"))
    G = int(os.environ.get("GS_G", "90"))
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10
    c = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(c, 0.0)
    s = DiscreteSwarmSolver(n_particles=P, max_generations=G + 5,
                            stall_generations=G + 5, random_state=1000)
    ctx = s._make_context(c)
    ctx.set_streams(numpy_stream_states(1000, P + 2))
    ctx.init(None, 0)
    ctx.step(3)
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(G)]
    fired = []
    for k in range(G):
        c0 = ctx.ctl()["two_opt_count"]
        ev[k][0].record(st)
        ctx.step(1)
        ev[k][1].record(st)
        torch.cuda.synchronize()
        fired.append(ctx.ctl()["two_opt_count"] > c0)
    ms = [a.elapsed_time(b) for a, b in ev]
    groups = {}
    for k in range(G):
        gen = 4 + k
        key = ("mut" if gen % 3 == 0 else "plain") + ("+2opt" if fired[k]
                                                      else "")
        groups.setdefault(key, []).append(ms[k])
    for key, v in sorted(groups.items()):
        print(f"{key:12s} n={len(v):3d} median {np.median(v):.4f} ms")
    ctx.close()


if __name__ == "__main__":
    main()
