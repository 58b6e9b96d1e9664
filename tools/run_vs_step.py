"""fit()'s run loop (dpso_run: graph batches + polling) against dpso_step on
the same swarm and seed, C2 shape: where does the end-to-end per-generation
time differ from the bench's per-step time?"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def make(seed, G):
    rng = np.random.default_rng(1000)
    pts = rng.random((1000, 2)) * 10.0
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    s = DiscreteSwarmSolver(n_particles=1024, max_generations=G,
                            stall_generations=G, random_state=seed)
    ctx = s._make_context(cost)
    ctx.set_streams(numpy_stream_states(seed, 1026))
    ctx.init(None, 0)
    torch.cuda.synchronize()
    return ctx


def main():
    G = 500
    for seed in (7, 1000):
        for mode in ("run", "step500", "step1", "bench_loop"):
            ctx = make(seed, G)
            t0 = time.perf_counter()
            if mode == "run":
                ctx.run()
            elif mode == "step500":
                ctx.step(G)
            elif mode == "step1":
                for _ in range(G):
                    ctx.step(1)
            else:
                # bench.py's timed loop: an L2 flush (untimed) between
                # CUDA-event-timed single steps
                flush = torch.empty(256 << 20, dtype=torch.uint8,
                                    device="cuda")
                ev = [(torch.cuda.Event(enable_timing=True),
                       torch.cuda.Event(enable_timing=True))
                      for _ in range(G)]
                for k in range(G):
                    flush.fill_(k & 0xFF)
                    ev[k][0].record()
                    ctx.step(1)
                    ev[k][1].record()
                torch.cuda.synchronize()
                tot = sum(a.elapsed_time(b) for a, b in ev)
                print(seed, "bench_loop events", f"{tot / G:.4f} ms/gen")
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            c = ctx.ctl()
            ctx.close()
            print(seed, mode, f"{dt * 1e3:.1f} ms", f"{dt / G * 1e3:.4f} ms/gen",
                  "2opt", c["two_opt_count"], "gens", c["gens_run"])


if __name__ == "__main__":
    main()
