"""Scene-scale parity of the device cost build (graph.py:
41-78): the office (816 viewpoints) and dense-obstacle bridge (500) scenes
of the scene-shaped bench configs, sampled rows against the Dijkstra oracle
(integer weights: the reference's admissible A* returns the same costs),
blocked pairs against unreachability."""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.gpu


def _row(args):
    from oracle import graph_oracle as G
    occ, w, vox, i = args
    d = G.dijkstra_all(occ, w, vox[i])
    return i, [d.get(tuple(int(c) for c in vox[j])) for j in range(len(vox))]


@pytest.mark.parametrize("name,rows", [("office", 32), ("bridge", 24)])
def test_scene_rows_vs_dijkstra(name, rows):
    import scenes
    from paper_1706_04399_b200 import build_cost_matrix
    occ, vox, w = scenes.scene(name)
    cost, virt, vcost = build_cost_matrix(occ, vox, w)
    n = len(vox)
    assert cost.shape == (n, n) and np.array_equal(cost, cost.T)
    assert not np.diag(cost).any()
    rng = np.random.default_rng(len(name))
    picks = sorted(int(i) for i in rng.choice(n, size=rows, replace=False))
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for i, d in ex.map(_row, [(occ, w, vox, i) for i in picks]):
            for j in range(n):
                if j == i:
                    continue
                if d[j] is None:
                    assert virt[i, j] and cost[i, j] == vcost, (name, i, j)
                else:
                    assert not virt[i, j] and cost[i, j] == d[j], (name, i, j)
    if virt.any():
        assert vcost == 1e3 * n * cost[~virt].max()
