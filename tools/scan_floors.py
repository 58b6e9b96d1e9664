"""Floors of the 2-opt scan at a swarm shape: the full scan against the
same kernel reduced to its row stream (DPSO_SCAN_STREAM_ONLY=1) and to the
row stream plus every pair's shared-memory gathers (=2), each timed with
CUDA events on the launching stream (dpso_step_timed's scan phase, only
generations where the scan ran).  Env: SF_N, SF_P, SF_GENS."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def main():
    n = int(os.environ.get("SF_N", "1000"))
    P = int(os.environ.get("SF_P", "1024"))
    G = int(os.environ.get("SF_GENS", "12"))
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10.0
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    out = {"n": n, "P": P}
    for name, val in (("full", None), ("stream_only", "1"),
                      ("stream_gathers", "2")):
        if val is None:
            os.environ.pop("DPSO_SCAN_STREAM_ONLY", None)
        else:
            os.environ["DPSO_SCAN_STREAM_ONLY"] = val
        s = DiscreteSwarmSolver(n_particles=P, max_generations=G + 4,
                                stall_generations=G + 4, random_state=7)
        ctx = s._make_context(cost)
        ctx.set_streams(numpy_stream_states(7, P + 2))
        ctx.init(None, 0)
        ctx.step_timed(2)  # warm-up
        ms = []
        for _ in range(G):
            c0 = ctx.ctl()["two_opt_count"]
            ph, cnt = ctx.step_timed(1)
            if cnt > c0:
                ms.append(float(ph[3]))
        ctx.close()
        out[name + "_ms"] = float(np.median(ms)) if ms else None
    os.environ.pop("DPSO_SCAN_STREAM_ONLY", None)
    pairs = n * (n - 1) // 2 * P
    out["pairs_per_launch"] = pairs
    for k in ("full", "stream_only", "stream_gathers"):
        if out.get(k + "_ms"):
            out[k + "_gpairs_per_s"] = pairs / out[k + "_ms"] / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
