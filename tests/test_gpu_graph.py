"""Device cost-matrix build vs the reference's build_graph (golden) and the
Dijkstra oracle."""
import numpy as np
import pytest

from conftest import GOLDEN
from oracle import graph_oracle as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def gg():
    return np.load(f"{GOLDEN}/golden_graph.npz")


def unpack(gg, name):
    dims = tuple(int(v) for v in gg[f"{name}__dims"])
    return np.unpackbits(gg[f"{name}__occ"])[:np.prod(dims)].reshape(
        dims).astype(bool)


@pytest.mark.parametrize("name", ["wall", "ablation", "sealed"])
def test_scene_matrices_bit_exact(pkg, gg, name):
    cost, virt, vcost = pkg.build_cost_matrix(
        unpack(gg, name), gg[f"{name}__vox"], gg[f"{name}__weights"])
    assert np.array_equal(cost, gg[f"{name}__cost"])
    assert np.array_equal(virt, gg[f"{name}__virtual"])
    assert vcost == gg[f"{name}__vcost"][0]


def test_random_grids_vs_reference_astar(pkg, gg):
    rows = gg["grid_pairs"]
    for seed in range(12):
        occ = np.unpackbits(gg[f"grid{seed}__occ"])[:4000].reshape(
            20, 20, 10).astype(bool)
        sub = rows[rows[:, 0] == seed]
        vox = [sub[0, 1:4]] + [r[4:7] for r in sub]
        w = sub[0, 7:10]
        # a goal may coincide with the source or be occupied-free only
        cost, virt, vcost = pkg.build_cost_matrix(occ, np.array(vox), w)
        integral = all(float(x).is_integer() for x in w)
        for k, r in enumerate(sub):
            want = r[10]
            got = vcost if virt[0, k + 1] else cost[0, k + 1]
            if not np.isfinite(want):
                assert virt[0, k + 1]
            elif integral:
                assert got == want, (seed, k)
            else:
                assert abs(got - want) <= 1e-12 * want, (seed, k)


def test_larger_grid_vs_oracle(pkg):
    rng = np.random.default_rng(3)
    occ = rng.random((40, 30, 12)) < 0.25
    free = np.argwhere(~occ)
    vox = free[rng.choice(len(free), size=24, replace=False)]
    for w in [(1.0, 1.0, 1.0), (2.0, 1.0, 3.0)]:
        cost, virt, vcost = pkg.build_cost_matrix(occ, vox, w)
        ocost, ovirt, ovc = G.build_cost(occ, vox, w)
        assert np.array_equal(cost, ocost)
        assert np.array_equal(virt, ovirt)
        assert vcost == ovc


def test_occupied_viewpoint_rejected(pkg):
    occ = np.zeros((5, 5, 5), dtype=bool)
    occ[2, 2, 2] = True
    with pytest.raises(ValueError, match="occupied"):
        pkg.build_cost_matrix(occ, [[0, 0, 0], [2, 2, 2]], (1, 1, 1))
