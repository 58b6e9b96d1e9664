"""Per-phase device time per generation over a whole solve, in segments
(default C2, 500 generations, segments of 50): how the step cost changes as
the swarm converges.  CUDA-event phase timing (dpso_step_timed).

    python tools/gen_profile.py [c2] [segment] > profiles/r02/gen_profile_c2.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    from paper_1706_04399_b200.solver import numpy_stream_states
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    seg = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    cfg = bench.CONFIGS[name]
    bench.RNG = cfg.get("rng", "numpy")  # as bench.py's main sets it
    cost, seed_tour = bench.make_matrix(cfg)
    P, G = cfg["P"], cfg["G"]
    params = bench.gpu_params(cfg, P, G, 7)
    if seed_tour is not None:
        params["seed_tour"] = seed_tour
    s = DiscreteSwarmSolver(**params)
    seed_body, n_seed = s._seed(cost.shape[0])
    ctx = s._make_context(cost)
    if params.get("rng", "numpy") == "numpy":
        ctx.set_streams(numpy_stream_states(7, P + 2))
    ctx.init(seed_body, n_seed)
    names = ["update", "mutation", "select", "two_opt_scan+apply",
             "two_opt_apply", "finalize"]
    out = []
    g = 0
    while g < G:
        b = min(seg, G - g)
        c0 = ctx.ctl()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        ms, cnt = ctx.step_timed(b)
        ev[1].record()
        torch.cuda.synchronize()
        c1 = ctx.ctl()
        out.append({"gens": [g, g + b],
                    "ms_per_gen": {k: round(float(v) / b, 4)
                                   for k, v in zip(names, ms)},
                    "wall_ms_per_gen": round(ev[0].elapsed_time(ev[1]) / b, 4),
                    "scans": cnt - c0["two_opt_count"],
                    "gbest": c1["gbest_fit"], "done": c1["done"]})
        print(json.dumps(out[-1]), flush=True)
        g += b
        if c1["done"]:
            break
    ctx.close()


if __name__ == "__main__":
    main()
