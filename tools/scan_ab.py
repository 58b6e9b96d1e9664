"""A/B timing of the 2-opt scan phase: the row-per-lane band scan against
the column-per-lane scan (DPSO_SCAN_BAND=0), at bench-config shapes.

Each variant: a swarm context at the shape, CUDA-event per-phase timing of
generations where the scan ran (dpso_step_timed phase 3 = scan + apply).

    python tools/scan_ab.py [c2 c3 c4 ...] > profiles/r02/scan_ab.json
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SHAPES = {
    "c1": (15, 32, "grid"),
    "c2": (1000, 1024, "euclid"),
    "c2i": (1000, 1024, "euclid_int"),
    "c3": (500, 16384, "grid"),
    "c4": (2000, 65536, "euclid"),
    "c4s": (2000, 4096, "euclid"),
    "n900": (900, 1024, "euclid"),
    "n800": (816, 1024, "euclid_int"),
}


def matrix(n, kind):
    rng = np.random.default_rng(n)
    if kind == "grid":
        side = int(math.ceil(math.sqrt(n)))
        idx = np.arange(n)
        pts = np.stack([idx % side, idx // side], 1).astype(float)
        return np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)
    pts = rng.random((n, 2))
    c = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    if kind == "euclid_int":
        c = np.floor(c * 1000.0)
    return c


def time_scan(n, P, cost, gens, env):
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    from paper_1706_04399_b200.solver import numpy_stream_states
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: v for k, v in env.items() if v is not None})
    try:
        G = gens + 8 + int(os.environ.get("AB_WARM", "0"))
        s = DiscreteSwarmSolver(n_particles=P, max_generations=G,
                                stall_generations=G, random_state=7,
                                rng="philox" if n * P > 50_000_000 else "numpy")
        ctx = s._make_context(cost)
        band = int(ctx.lib.dpso_scan_band(ctx.h))
        ctx.set_streams(numpy_stream_states(7, P + 2))
        ctx.init(None, 0)
        # AB_WARM: generations run first (a converged swarm has many more
        # near-tied deltas than random tours)
        ctx.step(int(os.environ.get("AB_WARM", "0")))
        ctx.step_timed(2)
        ms = []
        for _ in range(gens):
            c0 = ctx.ctl()["two_opt_count"]
            ph, _ = ctx.step_timed(1)
            if ctx.ctl()["two_opt_count"] > c0:
                ms.append(float(ph[3]))
        ctx.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    # mean over the generations where the scan ran (a mutating generation
    # runs the mutation-stream walk concurrently with the scan)
    return band, (float(np.mean(ms)) if ms else None)


def main():
    names = sys.argv[1:] or ["c2", "c3"]
    out = {}
    for name in names:
        n, P, kind = SHAPES[name]
        cost = matrix(n, kind)
        gens = int(os.environ.get("AB_GENS", "8"))
        rec = {"n": n, "P": P, "matrix": kind}
        variants = [("band", {}), ("column", {"DPSO_SCAN_BAND": "0"})]
        for st in os.environ.get("AB_STAGES", "").split(","):
            if st:
                variants.append(("band_stages" + st,
                                 {"DPSO_BAND_STAGES": st}))
        # AB_VARIANTS="tag:K=V,K=V;tag2:K=V": extra environment variants
        for spec in filter(None, os.environ.get("AB_VARIANTS", "").split(";")):
            tag, _, kvs = spec.partition(":")
            variants.append((tag, dict(kv.split("=", 1)
                                       for kv in kvs.split(",") if kv)))
        if os.environ.get("AB_PROBE"):
            variants.append(("band_stream_only", {"DPSO_BAND_PROBE": "1"}))
            variants.append(("band_consume_only", {"DPSO_BAND_PROBE": "2"}))
        for tag, env in variants:
            band, ms = time_scan(n, P, cost, gens, env)
            rec[tag] = {"scan_kind": band, "scan_apply_ms": ms}
        pairs = P * n * (n - 1) / 2
        for tag in [v[0] for v in variants]:
            ms = rec[tag]["scan_apply_ms"]
            if ms:
                rec[tag]["gpairs_per_s"] = pairs / ms / 1e6
                # int16/fp16 row stream: n rows of the particle, once each
                rec[tag]["row_stream_gbs"] = P * n * (2 * n + 16) / ms / 1e6
        out[name] = rec
        print(json.dumps({name: rec}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
