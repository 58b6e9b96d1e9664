"""2-opt scan time on a C2-shaped instance with blocked pairs (virtual
edges at 1e3 * n * max_finite, graph.py:63-78) against the plain one:
python tools/virtual_probe.py [frac_blocked]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1706_04399_b200 import DiscreteSwarmSolver  # noqa: E402
from paper_1706_04399_b200.solver import numpy_stream_states  # noqa: E402


def scan_ms(cost, P=1024, G=8):
    s = DiscreteSwarmSolver(n_particles=P, max_generations=G + 4,
                            stall_generations=G + 4, random_state=7)
    ctx = s._make_context(cost)
    ctx.set_streams(numpy_stream_states(7, P + 2))
    ctx.init(None, 0)
    ctx.step_timed(2)
    ms = []
    for _ in range(G):
        c0 = ctx.ctl()["two_opt_count"]
        ph, cnt = ctx.step_timed(1)
        if cnt > c0:
            ms.append(float(ph[3]))
    mode = ctx.lib.dpso_scan_mode(ctx.h)
    rows = ctx.lib.dpso_scan_rows_bytes(ctx.h)
    ctx.close()
    return (float(np.median(ms)) if ms else None), mode, rows


def main():
    frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
    n = 1000
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10
    c = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(c, 0.0)
    ci = np.floor(c * 20)  # integer scene-like costs
    out = {}
    for name, base in (("euclid", c), ("integer", ci)):
        out[name] = scan_ms(base)
        v = base.copy()
        blk = np.triu(rng.random((n, n)) < frac, 1)
        blk = blk | blk.T
        v[blk] = 1e3 * n * base.max()
        out[name + "_virtual"] = scan_ms(v)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
