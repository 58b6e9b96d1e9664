"""Synthetic inspection scenes for the scene-shaped bench configs (BASELINE
configs[1] "office-building-sized synthetic scene", configs[2]
"bridge-inspection-sized synthetic scene, dense obstacles") and the
cost-build parity tests.

A scene is an occupancy grid (True = occupied), axis weights and the
viewpoint voxels; ``scene_matrix`` turns it into the extended-TSP matrix
through the drop-in cost build (``build_cost_matrix``: graph.py:41-78
semantics, device SSSP).  The reference's path from a scene file to this
matrix is pipeline.py:43-51 (generate_viewpoints -> build_grid ->
build_graph); these generators stand in for generate_viewpoints/build_grid
(out of scope: SURVEY §2) with grids of the named sizes.

    python tools/scenes.py office|bridge   # build + cache tools/data/*.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DATA = os.path.join(HERE, "data")


def office_grid(nx=100, ny=48, nz=32):
    """Office floor (tools/bench_graph.py): boundary walls and floor, two
    pillars, a partition wall with a doorway, 24 desk blocks."""
    occ = np.zeros((nx, ny, nz), dtype=bool)
    occ[0, :, :] = occ[-1, :, :] = True
    occ[:, 0, :] = occ[:, -1, :] = True
    occ[:, :, 0] = True
    for cx, cy in ((30, 20), (70, 28)):
        occ[cx - 3:cx + 3, cy - 3:cy + 3, :] = True
    occ[50, 1:-1, 1:24] = True
    occ[50, 20:28, 1:18] = False
    rng = np.random.default_rng(7)
    for _ in range(24):
        x = int(rng.integers(3, nx - 10))
        y = int(rng.integers(3, ny - 8))
        occ[x:x + 6, y:y + 3, 1:4] = True
    return occ


def bridge_grid(nx=120, ny=40, nz=30, seed=11):
    """Girder bridge with dense clutter: ground, a deck slab, two rows of
    piers every 12 voxels, cross-bracing between them, scaffolding / debris
    boxes on the ground and under the deck."""
    occ = np.zeros((nx, ny, nz), dtype=bool)
    occ[:, :, 0] = True                          # ground
    occ[:, 5:35, 20:23] = True                   # deck
    occ[:, 5:7, 23:26] = occ[:, 33:35, 23:26] = True   # parapets
    for x in range(6, nx - 3, 12):               # piers
        for y in (10, 29):
            occ[x:x + 3, y:y + 3, 0:20] = True
    for x in range(6, nx - 15, 12):              # cross-bracing
        for k in range(12):
            z = 4 + k
            occ[x + k:x + k + 2, 10:13, z:z + 1] = True
            occ[x + k:x + k + 2, 29:32, z:z + 1] = True
        occ[x:x + 3, 12:30, 14:16] = True       # transverse beams
    rng = np.random.default_rng(seed)
    for _ in range(420):                         # scaffolding / debris
        x = int(rng.integers(1, nx - 6))
        y = int(rng.integers(1, ny - 6))
        z = int(rng.integers(1, 19))
        dx, dy, dz = (int(v) for v in rng.integers(1, 5, size=3))
        occ[x:x + dx, y:y + dy, z:z + dz] = True
    return occ


def surface_viewpoints(occ, n, seed, band=(1, 3)):
    """n free voxels at chamfer distance band[0]..band[1] from an occupied
    voxel (inspection standoff), spread by a fixed seed, sorted."""
    from scipy import ndimage
    d = ndimage.distance_transform_cdt(~occ, metric="chessboard")
    cand = np.argwhere((~occ) & (d >= band[0]) & (d <= band[1]))
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(cand), size=n, replace=False)
    return cand[np.sort(idx)].astype(np.int32)


def free_viewpoints(occ, n, seed):
    free = np.argwhere(~occ)
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(free), size=n, replace=False)
    return free[np.sort(idx)].astype(np.int32)


SCENES = {
    # C2-shaped: an office floor, 816 viewpoints, unit weights
    "office": dict(grid=office_grid, n=816, weights=(1.0, 1.0, 1.0),
                   vp=lambda occ: free_viewpoints(occ, 816, 816)),
    # C3-shaped: a bridge with dense obstacles, 500 viewpoints near the
    # structure, vertical moves twice as costly
    "bridge": dict(grid=bridge_grid, n=500, weights=(1.0, 1.0, 2.0),
                   vp=lambda occ: surface_viewpoints(occ, 500, 500)),
}


def scene(name):
    s = SCENES[name]
    occ = s["grid"]()
    vox = s["vp"](occ)
    return occ, vox, s["weights"]


def density(occ) -> float:
    return float(occ.mean())


def scene_matrix(name, allow_cache=True):
    """(cost, virtual, virtual_cost, meta): the device build when CUDA is
    available, else the cached build (tools/data/scene_<name>.npz, written
    by ``python tools/scenes.py <name>`` on a GPU box)."""
    occ, vox, w = scene(name)
    meta = {"scene": name, "grid": list(occ.shape), "voxels": int(occ.size),
            "rho": density(occ), "n": int(len(vox)), "weights": list(w)}
    path = os.path.join(DATA, f"scene_{name}.npz")
    try:
        import torch
        cuda = torch.cuda.is_available()
    except Exception:
        cuda = False
    if cuda:
        sys.path.insert(0, ROOT)
        from paper_1706_04399_b200 import build_cost_matrix
        cost, virt, vcost = build_cost_matrix(occ, vox, w)
        meta["source"] = "device build_cost_matrix"
        return cost, virt, vcost, meta
    if allow_cache and os.path.exists(path):
        z = np.load(path)
        meta["source"] = f"cache {os.path.relpath(path, ROOT)}"
        return z["cost"], z["virtual"], float(z["vcost"][0]), meta
    raise RuntimeError(f"scene {name}: no CUDA device and no cached build")


def main():
    name = sys.argv[1]
    cost, virt, vcost, meta = scene_matrix(name, allow_cache=False)
    os.makedirs(DATA, exist_ok=True)
    np.savez_compressed(os.path.join(DATA, f"scene_{name}.npz"), cost=cost,
                        virtual=virt, vcost=np.array([vcost]))
    print(meta, "virtual pairs", int(virt.sum() // 2),
          "max finite", float(cost[~virt].max()))


if __name__ == "__main__":
    main()
