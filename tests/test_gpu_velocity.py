"""Inertia w < 1 (solver.py:213-216: the kept velocity prefix is replayed
with the new transpositions): the device lists have no fixed bound - they
move to a larger buffer before they could overflow - so inertia close to 1
runs and matches the oracle bit for bit."""
import numpy as np
import pytest

from conftest import random_euclidean_matrix
from oracle import dpso_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


@pytest.mark.parametrize("w", [0.995, 0.9, 0.3])
def test_high_inertia_matches_oracle(pkg, w):
    rng = np.random.default_rng(int(w * 1000))
    cost = random_euclidean_matrix(20, rng)
    params = dict(n_particles=10, inertia=w, max_generations=300,
                  stall_generations=300, random_state=3)
    gpu = pkg.DiscreteSwarmSolver(**params).fit(cost)
    ref = O.OracleSolver(**params).fit(cost)
    assert gpu.best_tour_ == ref.best_tour_
    assert gpu.convergence_ == ref.convergence_
    assert gpu.n_generations_ == ref.n_generations_


def test_velocity_growth_through_step_and_state(pkg):
    # dpso_step batches grow the lists too; the swarm state matches the
    # oracle's after every 50 generations
    rng = np.random.default_rng(5)
    cost = random_euclidean_matrix(24, rng)
    params = dict(n_particles=8, inertia=0.99, max_generations=400,
                  stall_generations=400, random_state=8)
    s = pkg.DiscreteSwarmSolver(**params)
    from paper_1706_04399_b200.solver import numpy_stream_states
    ctx = s._make_context(cost)
    ref = O.OracleSolver(**params)
    ref.start(cost)
    try:
        ctx.set_streams(numpy_stream_states(params["random_state"], 10))
        ctx.init(None, 0)
        for _ in range(4):
            ctx.step(50)
            for _ in range(50):
                ref.generation()
            st = ctx.state()
            want = ref.state_
            assert st["x"].tolist() == want.x
            assert st["fit"].tolist() == want.fit
    finally:
        ctx.close()
