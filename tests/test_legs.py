"""Tour legs (voxel.py:112-172 A*, the paths graph.py:58-66 keeps): the
native A* returns the reference's waypoints and motion costs exactly
(golden vectors from the unmodified reference, tests/golden/
make_golden_legs.py), in both heuristic modes, blocked pairs as None.
Host code in libdpso.so: no GPU needed."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "golden_legs.json")) as fh:
        return json.load(fh)


def _occ(case):
    dims = tuple(case["dims"])
    bits = np.unpackbits(np.array(case["occ"], dtype=np.uint8))
    return bits[:int(np.prod(dims))].reshape(dims).astype(bool)


def test_wall_legs_all_pairs(pkg, golden):
    case = next(c for c in golden["cases"] if c["name"] == "wall")
    occ = _occ(case)
    n = len(case["vox"])
    tour = list(range(n)) + [0]
    got = pkg.tour_legs(occ, case["vox"], case["weights"], tour)
    want = {(i, j): (w, c) for i, j, w, c in case["legs"]}
    for key, val in got.items():
        w, c = want[key]
        assert val is not None
        assert [list(p) for p in val[0]] == w, key
        assert val[1] == c, key
    # every pair, in one batch
    from paper_1706_04399_b200.graph import _voxel_paths
    pairs = [list(case["vox"][i]) + list(case["vox"][j])
             for i, j, _, _ in case["legs"]]
    res = _voxel_paths(occ, pairs, case["weights"])
    for (i, j, w, c), r in zip(case["legs"], res):
        assert [list(p) for p in r[0]] == w and r[1] == c, (i, j)


def test_random_grids_both_modes(pkg, golden):
    for case in golden["cases"]:
        if not case["name"].startswith("grid"):
            continue
        occ = _occ(case)
        for a, b, w, c in case["pairs"]:
            r = pkg.shortest_path(occ, a, b, case["weights"],
                                  heuristic_mode=case["mode"])
            if w is None:
                assert r is None, (case["name"], a, b)
            else:
                assert [list(p) for p in r[0]] == w, (case["name"], a, b)
                assert r[1] == c, (case["name"], a, b)


def test_occupied_endpoint_and_trivial(pkg):
    from paper_1706_04399_b200.graph import OccupiedEndpointError
    occ = np.zeros((4, 4, 4), bool)
    occ[1, 1, 1] = True
    with pytest.raises(OccupiedEndpointError, match=r"start voxel \(1, 1, 1\)"):
        pkg.shortest_path(occ, (1, 1, 1), (0, 0, 0), (1.0, 1.0, 1.0))
    assert pkg.shortest_path(occ, (2, 2, 2), (2, 2, 2), (1.0, 1.0, 1.0)) == \
        (((2, 2, 2),), 0.0)
