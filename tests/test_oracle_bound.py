"""The bounded 2-opt scan's formulation (k_two_opt_bound.cu; restated as
oracle.dpso_oracle.bounded_exchange) returns the reference's
``_best_exchange`` result (solver.py:88-106) bit for bit, on CPU: random
tours (strong bound), 2-opt-optimal and nearly optimal tours (weak bound),
ties, asymmetric / negative / nonzero-diagonal / virtual-edge matrices and
extreme scales.  The GPU kernel is checked against the oracle in
tests/test_gpu_bound.py."""
import math

import numpy as np

from conftest import random_euclidean_matrix
from oracle import dpso_oracle as O


def grid(n):
    side = int(math.ceil(math.sqrt(n)))
    idx = np.arange(n)
    pts = np.stack([idx % side, idx // side], 1).astype(float)
    return np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)


def same(cost, body, tag, seeds=32):
    eb, ed = O.best_exchange(list(body), cost)
    bb, bd, _ = O.bounded_exchange(list(body), cost, seeds=seeds)
    assert [int(v) for v in bb] == [int(v) for v in eb], tag
    assert bd == ed, tag


def test_random_tours_all_kinds():
    rng = np.random.default_rng(1)
    for n in list(range(4, 30)) + [50, 97, 200]:
        mats = [random_euclidean_matrix(n, rng), grid(n),
                np.floor(random_euclidean_matrix(n, rng) * 100.0),
                rng.normal(size=(n, n))]
        a = random_euclidean_matrix(n, rng) * (1 + rng.random((n, n)))
        np.fill_diagonal(a, 0.0)
        mats.append(a)
        dg = random_euclidean_matrix(n, rng)
        np.fill_diagonal(dg, -3.0)
        mats.append(dg)
        for m, cost in enumerate(mats):
            for _ in range(3):
                same(cost, rng.permutation(n), (n, m))


def test_pruning_is_strong_on_random_tours():
    rng = np.random.default_rng(2)
    n = 300
    cost = random_euclidean_matrix(n, rng)
    for _ in range(5):
        body = list(rng.permutation(n))
        _, _, ev = O.bounded_exchange(body, cost)
        assert ev < 0.01 * n * (n - 1) / 2
        same(cost, body, "random")


def test_optimal_and_nearly_optimal_tours():
    rng = np.random.default_rng(3)
    for n, cost in ((40, grid(40)), (80, random_euclidean_matrix(80, rng)),
                    (120, grid(120))):
        nn, _ = O.nearest_neighbor_two_opt(cost)
        base = list(nn[:-1])
        same(cost, base, ("opt", n))
        for swaps in (1, 2, 5, 30):
            b = list(base)
            for _ in range(swaps):
                i, j = rng.integers(0, n, 2)
                b[i], b[j] = b[j], b[i]
            same(cost, b, ("near", n, swaps))


def test_virtual_edges_scales_ties():
    rng = np.random.default_rng(4)
    n = 90
    v = np.floor(random_euclidean_matrix(n, rng) * 100.0)
    mask = np.triu(rng.random((n, n)) < 0.03, 1)
    mask = mask | mask.T
    v[mask] = 1e3 * n * v[~mask].max()
    for mul in (1.0, 1e-200, 1e-6, 1e9, 1e250):
        for _ in range(3):
            same(v * mul, rng.permutation(n), ("virtual", mul))
            same(random_euclidean_matrix(n, rng) * mul, rng.permutation(n),
                 ("scale", mul))
    same(grid(100) / 3.0, rng.permutation(100), "lattice")
    same(np.zeros((30, 30)), rng.permutation(30), "zeros")
    for seeds in (1, 2, 8):
        same(grid(64), rng.permutation(64), ("seeds", seeds), seeds=seeds)


def test_swarm_tours_from_a_solve():
    # the tours the solver actually scans (oracle swarm after a few
    # generations), N = 200
    rng = np.random.default_rng(5)
    cost = random_euclidean_matrix(200, rng)
    s = O.OracleSolver(n_particles=12, max_generations=8, stall_generations=8,
                       random_state=3).start(cost)
    for _ in range(6):
        s.generation()
        for body in s.state_.x:
            same(cost, body, "swarm")
