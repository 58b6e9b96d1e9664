"""Golden ``inspectour plan`` outputs of the UNMODIFIED reference CLI
(cli.py:149-173: tour.json, convergence.csv, cost_matrix.txt), with the
inputs the drop-in path consumes, so a GPU test can swap this package's
``build_graph`` and ``DiscreteSwarmSolver`` into the same pipeline and
compare the files byte for byte.

Run in the build container only (``/root/reference`` does not exist on the
GPU box)::

    python tests/golden/make_golden_plan.py   # -> golden_plan.json

Scenes: pkg/scenes/wall.json (the reference's own, N=15) and
tests/golden/scenes/piers.json (two surfaces, five obstacles, non-unit z
weight, N=76); heuristics "admissible" and "paper"; solver flags: CLI
defaults except --generations / --particles below (every seed-fraction,
mutation and 2-opt default kept).
"""
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))

from inspectour.cli import main as cli_main  # noqa: E402
from inspectour.scene import load_scene  # noqa: E402
from inspectour.viewpoints import (boustrophedon_tour,  # noqa: E402
                                   generate_viewpoints)
from inspectour.voxel import build_grid  # noqa: E402

RUNS = [
    ("wall", os.path.join(REF, "scenes", "wall.json"), "admissible",
     ["--generations", "200"]),
    ("wall", os.path.join(REF, "scenes", "wall.json"), "paper",
     ["--generations", "200", "--seed", "3"]),
    ("piers", os.path.join(HERE, "scenes", "piers.json"), "admissible",
     ["--generations", "60", "--particles", "48", "--seed", "5"]),
    ("piers", os.path.join(HERE, "scenes", "piers.json"), "paper",
     ["--generations", "40", "--particles", "32", "--seed", "9"]),
]


def main():
    out = {"runs": []}
    for name, path, heur, flags in RUNS:
        scene = load_scene(path)
        plan = generate_viewpoints(scene)
        grid = build_grid(scene)
        with tempfile.TemporaryDirectory() as d:
            argv = ["plan", "--scene", path, "--out", d, "--heuristic",
                    heur] + flags
            assert cli_main(argv) == 0
            files = {f: open(os.path.join(d, f)).read()
                     for f in ("tour.json", "convergence.csv",
                               "cost_matrix.txt")}
        out["runs"].append({
            "scene": name, "heuristic": heur, "argv": argv[5:],
            "weights": list(scene.axis_weights),
            "viewpoints": [{"id": vp.id,
                            "position": [float(c) for c in vp.position],
                            "orientation": [float(c) for c in vp.orientation],
                            "surface_index": vp.surface_index}
                           for vp in plan.viewpoints],
            "seed_tour": [int(v) for v in boustrophedon_tour(plan)],
            "grid": {"dims": list(grid.dims),
                     "origin": [float(c) for c in grid.origin],
                     "voxel_size": float(grid.voxel_size),
                     "occ": np.packbits(grid.occupancy.ravel()).tolist()},
            "files": files})
        print(name, heur, len(plan.viewpoints), flush=True)
    with open(os.path.join(HERE, "golden_plan.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
