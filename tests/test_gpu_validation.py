"""fit()'s input validation (solver.py:139-162, 169-172) through the GPU
path: the reference's own cases (test_solver.py:39-49, 222-226) plus
non-finite matrices, host and device, and the island API."""
import numpy as np
import pytest

from conftest import random_euclidean_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


def test_rejects_bad_matrix(pkg):
    with pytest.raises(ValueError, match="must be square"):
        pkg.DiscreteSwarmSolver().fit(np.zeros((3, 2)))


def test_rejects_bad_params(pkg):
    c = np.zeros((3, 3))
    for kw, msg in ((dict(n_particles=2), "n_particles must be >= 3"),
                    (dict(inertia=1.5), "inertia must be in"),
                    (dict(mutation_period=0), "mutation_period must be"),
                    (dict(max_generations=0), "max_generations must be"),
                    (dict(seed_fraction=2.0), "seed_fraction must be")):
        with pytest.raises(ValueError, match=msg):
            pkg.DiscreteSwarmSolver(**kw).fit(c)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_rejects_non_finite(pkg, bad):
    import torch
    c = random_euclidean_matrix(40, np.random.default_rng(3))
    c[7, 11] = bad
    with pytest.raises(ValueError, match="cost matrix must be finite"):
        pkg.DiscreteSwarmSolver(n_particles=8).fit(c)
    with pytest.raises(ValueError, match="cost matrix must be finite"):
        pkg.DiscreteSwarmSolver(n_particles=8).fit(torch.from_numpy(c).cuda())
    with pytest.raises(ValueError, match="cost matrix must be finite"):
        pkg.IslandSolver(devices=["cuda:0"], n_particles=8).fit(c)


def test_invalid_seed_tour_rejected(pkg):
    c = random_euclidean_matrix(5, np.random.default_rng(14))
    with pytest.raises(ValueError, match="seed_tour is not a tour"):
        pkg.DiscreteSwarmSolver(seed_tour=(0, 1, 2, 0), random_state=0).fit(c)


def test_matrix_error_before_seed_tour_error(pkg):
    # the reference checks the matrix before the seed tour
    c = random_euclidean_matrix(5, np.random.default_rng(14))
    c[0, 1] = np.nan
    with pytest.raises(ValueError, match="finite"):
        pkg.DiscreteSwarmSolver(seed_tour=(0, 1, 2, 0), random_state=0).fit(c)


def test_single_node(pkg):
    s = pkg.DiscreteSwarmSolver(random_state=0).fit(np.zeros((1, 1)))
    assert s.best_tour_ == (0, 0)
    assert s.best_fitness_ == 0.0
    assert s.convergence_ == [0.0]
