"""Pin the cost-matrix oracle (oracle/graph_oracle.py) against the reference's
build_graph / shortest_path outputs (tests/golden/make_golden_graph.py)."""
import numpy as np
import pytest

from conftest import GOLDEN
from oracle import graph_oracle as G


@pytest.fixture(scope="module")
def gg():
    return np.load(f"{GOLDEN}/golden_graph.npz")


def unpack(gg, name):
    dims = tuple(int(v) for v in gg[f"{name}__dims"])
    occ = np.unpackbits(gg[f"{name}__occ"])[:np.prod(dims)].reshape(dims)
    return occ.astype(bool)


@pytest.mark.parametrize("name", ["wall", "ablation", "sealed"])
def test_scene_matrices(gg, name):
    occ = unpack(gg, name)
    cost, virt, vcost = G.build_cost(occ, gg[f"{name}__vox"],
                                     tuple(gg[f"{name}__weights"]))
    assert np.array_equal(cost, gg[f"{name}__cost"])
    assert np.array_equal(virt, gg[f"{name}__virtual"])
    assert vcost == gg[f"{name}__vcost"][0]


def test_random_grid_pairs(gg):
    rows = gg["grid_pairs"]
    for seed in range(12):
        occ = np.unpackbits(gg[f"grid{seed}__occ"])[:4000].reshape(20, 20, 10)
        sub = rows[rows[:, 0] == seed]
        src = tuple(int(v) for v in sub[0, 1:4])
        w = tuple(sub[0, 7:10])
        d = G.dijkstra_all(occ.astype(bool), w, src)
        integral = all(float(x).is_integer() for x in w)
        for r in sub:
            got = d.get(tuple(int(v) for v in r[4:7]), np.inf)
            if integral or not np.isfinite(r[10]):
                assert got == r[10], (seed, r)
            else:
                # non-integer weights: A* keeps the first path its
                # (f, g, voxel) order settles, whose fp sum can exceed the
                # fp minimum (Dijkstra) by an ulp
                assert got <= r[10] and abs(got - r[10]) <= 1e-12 * r[10]
