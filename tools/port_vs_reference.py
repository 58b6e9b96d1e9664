"""The oracle port (oracle/dpso_oracle.py, the `--impl reference` arm of
bench.py) against the UNMODIFIED reference solver, same container, same
instance and seeds: identical results, and the rate each reaches on one
core.  Runs where /root/reference exists (the build container); writes
profiles/r02/port_vs_reference.json, which bench.py's reference line cites.

    python tools/port_vs_reference.py [n] [P] [G] [reps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from inspectour.solver import DiscreteSwarmSolver as Ref  # noqa: E402
from oracle.dpso_oracle import OracleSolver as Port  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    n, P, G, reps = (a + [1000, 32, 8, 2][len(a):])[:4]
    rng = np.random.default_rng(1000)
    pts = rng.random((n, 2)) * 10.0
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    np.fill_diagonal(cost, 0.0)
    out = {"n": n, "P": P, "generations": G, "reps": reps, "runs": []}
    tr, tp = [], []
    for r in range(reps):
        kw = dict(n_particles=P, max_generations=G, stall_generations=G,
                  random_state=100 + r)
        t0 = time.perf_counter()
        ref = Ref(**kw).fit(cost)
        t1 = time.perf_counter()
        port = Port(**kw).fit(cost)
        t2 = time.perf_counter()
        same = (list(ref.best_tour_) == list(port.best_tour_)
                and list(ref.convergence_) == list(port.convergence_))
        tr.append(t1 - t0)
        tp.append(t2 - t1)
        out["runs"].append({"seed": 100 + r, "identical": same,
                            "reference_s": t1 - t0, "port_s": t2 - t1})
    work = P * G
    out["reference_rate"] = work * reps / sum(tr)
    out["port_rate"] = work * reps / sum(tp)
    out["unit"] = "particle-iterations/s, one core, fit() wall time"
    out["identical"] = all(r["identical"] for r in out["runs"])
    path = os.path.join(ROOT, "profiles", "r02", "port_vs_reference.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
