"""Golden waypoint legs (voxel.py:112-172 shortest_path, the paths
graph.py:58-66 stores as TourGraph.legs), produced by running the UNMODIFIED
reference here: ``python tests/golden/make_golden_legs.py`` ->
golden_legs.json.

* wall.json: every pair i < j (the legs the reference keeps for its graph),
  admissible mode;
* random 20x20x10 grids, 20% obstacles (test_acceptance.py:120-144 shape):
  12 (start, goal) pairs per grid, admissible and paper modes, integer and
  non-integer axis weights; blocked pairs recorded as null.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))

from inspectour.scene import load_scene  # noqa: E402
from inspectour.viewpoints import generate_viewpoints  # noqa: E402
from inspectour.voxel import VoxelGrid, build_grid, shortest_path  # noqa: E402


def main():
    out = {"cases": []}
    scene = load_scene(os.path.join(REF, "scenes", "wall.json"))
    plan = generate_viewpoints(scene)
    grid = build_grid(scene)
    vox = [grid.point_to_voxel(vp.position) for vp in plan.viewpoints]
    legs = []
    for i in range(len(vox)):
        for j in range(i + 1, len(vox)):
            p = shortest_path(grid, vox[i], vox[j], scene.axis_weights)
            legs.append([i, j, None if p is None else
                         [list(map(int, w)) for w in p.waypoints],
                         None if p is None else p.motion_cost])
    out["cases"].append({
        "name": "wall", "dims": list(grid.dims),
        "occ": np.packbits(grid.occupancy.ravel()).tolist(),
        "weights": list(scene.axis_weights), "mode": "admissible",
        "vox": [list(map(int, v)) for v in vox], "legs": legs})
    for seed in range(8):
        rng = np.random.default_rng(100 + seed)
        dims = (20, 20, 10)
        occ = rng.random(dims) < 0.20
        free = np.argwhere(~occ)
        weights = (tuple(float(w) for w in rng.integers(1, 4, size=3))
                   if seed < 5 else (0.3, 1.7, 2.9))
        g = VoxelGrid(dims, np.zeros(3), 1.0, occ)
        for mode in ("admissible", "paper"):
            pairs = []
            for _ in range(12):
                a = free[rng.integers(len(free))]
                b = free[rng.integers(len(free))]
                p = shortest_path(g, tuple(a), tuple(b), weights,
                                  heuristic_mode=mode)
                pairs.append([list(map(int, a)), list(map(int, b)),
                              None if p is None else
                              [list(map(int, w)) for w in p.waypoints],
                              None if p is None else p.motion_cost])
            out["cases"].append({
                "name": f"grid{seed}_{mode}", "dims": list(dims),
                "occ": np.packbits(occ.ravel()).tolist(),
                "weights": list(weights), "mode": mode, "pairs": pairs})
    with open(os.path.join(HERE, "golden_legs.json"), "w") as fh:
        json.dump(out, fh)
    print(len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
