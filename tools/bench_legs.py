"""Tour legs on the office-sized grid (tools/bench_graph.py's synthetic
100x48x32 office, 816 viewpoints): the native A* (tour_legs, all host
cores) for the 816 edges of a tour, against the reference's Python A*
timed on a few of the same legs (the per-leg rate x 816 is the estimate).
Run where the reference is importable (this container):
python tools/bench_legs.py [ref_sample]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

from bench_graph import office_grid, viewpoints  # noqa: E402
import paper_1706_04399_b200 as pkg  # noqa: E402


def main():
    sample = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    occ = office_grid()
    vox = viewpoints(occ, 816)
    n = len(vox)
    tour = list(np.random.default_rng(3).permutation(n)) + []
    tour = tour + [tour[0]]
    w = (1.0, 1.0, 1.0)
    t = time.perf_counter()
    legs = pkg.tour_legs(occ, vox, w, tour)
    native = time.perf_counter() - t
    out = {"legs": len(legs), "native_s": native, "cores": os.cpu_count()}
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        sys.path.insert(0, ref)
        from inspectour.voxel import VoxelGrid, shortest_path
        g = VoxelGrid(occ.shape, np.zeros(3), 1.0, occ)
        keys = list(legs)[:sample]
        t = time.perf_counter()
        same = True
        for i, j in keys:
            p = shortest_path(g, tuple(vox[i]), tuple(vox[j]), w)
            mine = legs[(i, j)]
            same &= (p is None and mine is None) or (
                mine is not None and tuple(map(tuple, p.waypoints)) == mine[0]
                and p.motion_cost == mine[1])
        per = (time.perf_counter() - t) / len(keys)
        out.update(reference_s_per_leg=per,
                   reference_est_s=per * len(legs), sample_identical=same)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
