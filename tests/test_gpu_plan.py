"""The drop-in on the reference's own pipeline: ``inspectour plan`` with
this package's ``build_graph`` (device SSSP cost build, or the native A*
in "paper" mode; lazy legs) and ``DiscreteSwarmSolver`` swapped in writes
tour.json, convergence.csv and cost_matrix.txt byte for byte as the
unmodified reference CLI did (tests/golden/make_golden_plan.py; the output
shape of the reference's test_cli.py:44-65)."""
import os

import pytest

from conftest import GOLDEN, load_golden
from plan_restated import Grid, Plan, run_plan

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


def _runs():
    if not os.path.exists(os.path.join(GOLDEN, "golden_plan.json")):
        return []
    return load_golden("golden_plan.json")["runs"]


@pytest.mark.parametrize("rec", _runs(),
                         ids=lambda r: f"{r['scene']}-{r['heuristic']}")
def test_plan_outputs_byte_identical(pkg, rec, tmp_path):
    files = run_plan(pkg, rec, str(tmp_path))
    for name in ("cost_matrix.txt", "convergence.csv", "tour.json"):
        assert files[name] == rec["files"][name], (rec["scene"], name)


def test_build_graph_infeasible_viewpoint(pkg):
    from paper_1706_04399_b200.errors import InfeasibleViewpointError
    rec = _runs()[0]
    grid = Grid(rec["grid"])
    plan = Plan(rec["viewpoints"])
    idx = grid.point_to_voxel(plan.viewpoints[2].position)
    occ = grid.occupancy.copy()
    occ[idx] = True
    grid.occupancy = occ
    with pytest.raises(InfeasibleViewpointError,
                       match=rf"viewpoint {plan.viewpoints[2].id} maps to "
                             rf"occupied voxel"):
        pkg.build_graph(plan, grid, tuple(rec["weights"]))


def test_lazy_legs_mapping(pkg):
    rec = _runs()[0]
    g = pkg.build_graph(Plan(rec["viewpoints"]), Grid(rec["grid"]),
                        tuple(rec["weights"]))
    n = g.n_nodes
    assert len(g.legs) == sum(1 for i in range(n) for j in range(i + 1, n)
                              if not g.virtual[i, j])
    p = g.leg(0, 3)
    q = g.leg(3, 0)
    assert p.waypoints == tuple(reversed(q.waypoints))
    assert p.motion_cost == g.cost[0, 3]
    assert g.leg(2, 2) is None
