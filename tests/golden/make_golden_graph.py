"""Golden vectors for the cost-matrix build (graph.py:41-78, voxel.py:112-172),
produced by running the UNMODIFIED reference here:
``python tests/golden/make_golden_graph.py`` -> golden_graph.npz.

* scene instances (wall.json; the 36-node ablation scene; the sealed-wall
  scene of test_acceptance.py:288-292): occupancy grid, viewpoint voxels,
  axis weights, the reference's cost matrix, virtual mask, virtual cost;
* random grids (test_acceptance.py:120-144 shape: 20x20x10, 20% obstacles,
  integer weights 1..3, plus one non-integer weight set): shortest_path
  costs for sampled (start, goal) pairs, inf when blocked.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from conftest import make_scene  # noqa: E402
from inspectour.graph import build_graph  # noqa: E402
from inspectour.scene import load_scene  # noqa: E402
from inspectour.viewpoints import generate_viewpoints  # noqa: E402
from inspectour.voxel import VoxelGrid, build_grid, shortest_path  # noqa: E402


def scene_case(scene):
    plan = generate_viewpoints(scene)
    grid = build_grid(scene)
    g = build_graph(plan, grid, scene.axis_weights)
    vox = np.array([grid.point_to_voxel(vp.position) for vp in plan.viewpoints],
                   dtype=np.int32)
    return dict(occ=np.packbits(grid.occupancy.ravel()),
                dims=np.array(grid.dims, dtype=np.int32), vox=vox,
                weights=np.array(scene.axis_weights, dtype=float),
                cost=np.array(g.cost), virtual=np.array(g.virtual),
                vcost=np.array([g.virtual_cost]))


def main():
    out = {}
    scenes = {
        "wall": load_scene(os.path.join(REF, "scenes", "wall.json")),
        "ablation": make_scene(rows=6, cols=6, voxel_size=0.4,
                               vehicle_radius=0.1,
                               obstacles=[((3.3, 5.0, 0.0), (3.5, 7.4, 3.6))]),
        "sealed": make_scene(rows=1, cols=3, voxel_size=0.4,
                             obstacles=[((1.7, 0.0, 0.0), (1.9, 10.0, 6.0))]),
    }
    for name, sc in scenes.items():
        for k, v in scene_case(sc).items():
            out[f"{name}__{k}"] = v
    rows = []
    for seed in range(12):
        rng = np.random.default_rng(seed)
        dims = (20, 20, 10)
        occ = rng.random(dims) < 0.20
        free = np.argwhere(~occ)
        if seed < 10:
            weights = tuple(float(w) for w in rng.integers(1, 4, size=3))
        else:
            weights = (0.3, 1.7, 2.9) if seed == 10 else (1.1, 0.7, 0.35)
        grid = VoxelGrid(dims, np.zeros(3), 1.0, occ)
        src = free[rng.integers(len(free))]
        goals = free[rng.choice(len(free), size=12, replace=False)]
        for gl in goals:
            p = shortest_path(grid, tuple(src), tuple(gl), weights)
            rows.append((seed, *src, *gl, *weights,
                         np.inf if p is None else p.motion_cost))
        out[f"grid{seed}__occ"] = np.packbits(occ.ravel())
    out["grid_pairs"] = np.array(rows, dtype=float)
    np.savez_compressed(os.path.join(HERE, "golden_graph.npz"), **out)
    print({k: v.shape for k, v in out.items() if k.endswith("cost")},
          len(rows))


if __name__ == "__main__":
    main()
