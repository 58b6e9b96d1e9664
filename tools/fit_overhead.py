"""Where the wall time of one public ``DiscreteSwarmSolver.fit`` goes at a
bench shape (default C2: N=1000, P=1024, 500 generations): parameter and
matrix checks, the matrix upload, context creation (workspace, plan, graph
capture), the numpy stream states, init, the generation loop, the result
read-back and close.  Host-timed with a device sync after each phase.

    python tools/fit_overhead.py [c2|c2s|c3] > profiles/r02/fit_overhead_c2.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    from paper_1706_04399_b200.solver import (SwarmContext,
                                              numpy_stream_states)
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = bench.CONFIGS[name]
    bench.RNG = cfg.get("rng", "numpy")  # as bench.py's main sets it
    cost, seed_tour = bench.make_matrix(cfg)
    P, G = cfg["P"], cfg["G"]
    params = bench.gpu_params(cfg, P, G, 7)
    if seed_tour is not None:
        params["seed_tour"] = seed_tour
    DiscreteSwarmSolver(**params).fit(cost)  # warm-up (module, pools, JIT)
    out = {"config": name, "n": cfg["n"], "P": P, "G": G}
    reps = []
    for _ in range(3):
        ph = {}
        torch.cuda.synchronize()
        t_all = time.perf_counter()

        def mark(key, t):
            torch.cuda.synchronize()
            now = time.perf_counter()
            ph[key] = round((now - t) * 1e3, 3)
            return now

        t = time.perf_counter()
        s = DiscreteSwarmSolver(**params)
        s._check_params()
        # fit()'s path: shape check on the host, upload, finiteness on the
        # device
        cost_t, ld = s._upload_cost(cost)
        t = mark("checks_and_h2d_ms", t)
        n = cost_t.shape[0]
        ctx = SwarmContext(s._params(), n, cost_t, ld)
        t = mark("context_ms", t)
        seed_body, n_seed = s._seed(n)
        if s.rng == "numpy":
            st = numpy_stream_states(s.random_state, P + 2)
            t = mark("stream_states_ms", t)
            ctx.set_streams(st)
            t = mark("set_streams_ms", t)
        ctx.init(seed_body, n_seed)
        t = mark("init_ms", t)
        gens = ctx.run()
        t = mark("run_ms", t)
        ctx.result()
        t = mark("result_ms", t)
        ctx.close()
        t = mark("close_ms", t)
        ph["total_ms"] = round((time.perf_counter() - t_all) * 1e3, 3)
        ph["generations"] = gens
        ph["run_ms_per_gen"] = round(ph["run_ms"] / gens, 4)
        reps.append(ph)
    out["reps"] = reps
    print(json.dumps(out))


if __name__ == "__main__":
    main()
