"""GPU parity of the bounded 2-opt scan (k_two_opt_bound.cu) against the
oracle's ``_best_exchange`` (solver.py:88-106): the pair bound
delta(i, j) >= -(h_i + h_j) prunes pairs, the rest are evaluated with the
reference expression in fp64, particles with a weak bound go to the band
scan.  Random tours (strong bound), 2-opt-optimal and nearly optimal tours
(weak bound, band fallback), ties, asymmetric / negative / virtual-edge
matrices, a forced small row list, and whole solves."""
import math

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


def ctx_query(pkg, cost, fn):
    s = pkg.DiscreteSwarmSolver(n_particles=4)
    ctx = s._make_context(cost)
    try:
        return int(getattr(ctx.lib, fn)(ctx.h))
    finally:
        ctx.close()


def check(pkg, cost, tours, tag, sample=None, rng=None):
    new, delta = pkg.best_exchange_batch(cost, tours)
    idx = range(len(tours))
    if sample is not None and len(tours) > sample:
        idx = rng.choice(len(tours), size=sample, replace=False)
    for p in idx:
        eb, ed = O.best_exchange([int(v) for v in tours[p]], cost)
        assert [int(v) for v in new[p]] == [int(v) for v in eb], (tag, int(p))
        assert float(delta[p]) == ed, (tag, int(p))
    assert (np.sort(new, axis=1) == np.arange(cost.shape[0])).all(), tag


def perms(rng, P, n):
    return rng.permuted(np.tile(np.arange(n, dtype=np.int32), (P, 1)), axis=1)


def grid(n):
    side = int(math.ceil(math.sqrt(n)))
    idx = np.arange(n)
    pts = np.stack([idx % side, idx // side], 1).astype(float)
    return np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)


def near_optimal(rng, cost, P, swaps):
    """2-opt-optimal NN tour with a few random transpositions per copy: a
    weak bound (many rows can still improve a little)."""
    nn, _ = O.nearest_neighbor_two_opt(cost)
    base = np.array(nn[:-1], dtype=np.int32)
    out = np.tile(base, (P, 1))
    n = len(base)
    for p in range(P):
        for _ in range(swaps[p % len(swaps)]):
            i, j = rng.integers(0, n, 2)
            out[p, i], out[p, j] = out[p, j], out[p, i]
    return out


def test_bound_selected(pkg, monkeypatch):
    rng = np.random.default_rng(1)
    assert ctx_query(pkg, grid(100), "dpso_scan_bound") == 1
    assert ctx_query(pkg, random_euclidean_matrix(100, rng),
                     "dpso_scan_bound") == 1
    inf = random_euclidean_matrix(100, rng)
    inf[3, 7] = np.inf  # non-finite entries: the full scan
    assert ctx_query(pkg, inf, "dpso_scan_bound") == 0
    monkeypatch.setenv("DPSO_BOUND", "0")
    assert ctx_query(pkg, grid(100), "dpso_scan_bound") == 0


@pytest.fixture(params=["256", "128"])
def threads(request, monkeypatch):
    # CTA width: 256 threads (32 seed rows) for small swarms, 128 (16) for
    # large ones; both forced here
    monkeypatch.setenv("DPSO_BOUND_NT", request.param)
    return request.param


@pytest.mark.parametrize("kind", ["euclid", "grid", "int"])
def test_bound_random_tours(pkg, kind, threads):
    rng = np.random.default_rng(3)
    for n in list(range(4, 40)) + [63, 64, 65, 100, 257, 511, 1000]:
        if kind == "grid":
            cost = grid(n)
        else:
            cost = random_euclidean_matrix(n, rng)
            if kind == "int":
                cost = np.floor(cost * 100.0)
        check(pkg, cost, perms(rng, 16, n), (kind, n))


def test_bound_large_n(pkg):
    rng = np.random.default_rng(5)
    for n in (2000, 2548, 2900):
        cost = random_euclidean_matrix(n, rng)
        check(pkg, cost, perms(rng, 8, n), ("large", n), 4, rng)


def test_bound_ties_and_optimal_tours(pkg, threads):
    rng = np.random.default_rng(7)
    for n in (16, 49, 100, 300):
        cost = grid(n)
        # 2-opt-optimal tours: no improving pair (weak bound: band fallback)
        nn, _ = O.nearest_neighbor_two_opt(cost)
        check(pkg, cost, np.array([nn[:-1]] * 3, dtype=np.int32), ("opt", n))
        check(pkg, cost, near_optimal(rng, cost, 24, [0, 1, 2, 5, 40]),
              ("near", n))


def test_bound_near_optimal_euclid(pkg, threads):
    rng = np.random.default_rng(9)
    for n in (50, 200, 600):
        cost = random_euclidean_matrix(n, rng)
        check(pkg, cost, near_optimal(rng, cost, 32, [0, 1, 2, 3, 8, 100]),
              ("near-euclid", n))


def test_bound_scales(pkg):
    rng = np.random.default_rng(11)
    for n, mul in ((200, 1.0), (200, 1e-6), (200, 1e9), (300, 3.7),
                   (120, 1e-200), (120, 1e250)):
        cost = random_euclidean_matrix(n, rng) * mul
        check(pkg, cost, perms(rng, 16, n), ("scale", n, mul))
    cost = np.floor(random_euclidean_matrix(300, rng) * 1e7)
    check(pkg, cost, perms(rng, 16, 300), "wide-int")
    check(pkg, np.zeros((40, 40)), perms(rng, 4, 40), "zeros")
    check(pkg, grid(144) / 3.0, perms(rng, 12, 144), "lattice")


def test_bound_asymmetric_negative_virtual(pkg, threads):
    rng = np.random.default_rng(17)
    n = 257
    c = random_euclidean_matrix(n, rng) * (1 + rng.random((n, n)))
    np.fill_diagonal(c, 0.0)
    check(pkg, c, perms(rng, 12, n), "asym")
    check(pkg, np.floor(c * 50.0), perms(rng, 12, n), "asym-int")
    neg = rng.normal(size=(n, n))
    check(pkg, neg, perms(rng, 12, n), "normal")
    check(pkg, np.round(neg * 100.0), perms(rng, 12, n), "normal-int")
    # nonzero diagonal: the bound uses off-diagonal minima only
    d = random_euclidean_matrix(n, rng)
    np.fill_diagonal(d, -5.0)
    check(pkg, d, perms(rng, 12, n), "diag")
    v = np.floor(random_euclidean_matrix(n, rng) * 100.0)
    mask = np.triu(rng.random((n, n)) < 0.02, 1)
    mask = mask | mask.T
    v[mask] = 1e3 * n * v[~mask].max()
    check(pkg, v, perms(rng, 12, n), "virtual-int")
    ve = random_euclidean_matrix(n, rng)
    ve[mask] = 1e3 * n * ve[~mask].max()
    check(pkg, ve, perms(rng, 12, n), "virtual")
    check(pkg, ve, near_optimal(rng, ve, 12, [0, 2, 9]), "virtual-near")


@pytest.mark.parametrize("peel", ["0", "3", "64"])
@pytest.mark.parametrize("rmax", ["32", "40", "100"])
def test_bound_small_row_list(pkg, rmax, peel, threads, monkeypatch):
    # a small row-list capacity makes the kernel peel rows of largest h
    # (paired with every row they reach) and, past the peel limit, send
    # the particle to the band scan: the two kernels' results interleave
    monkeypatch.setenv("DPSO_BOUND_RMAX", rmax)
    monkeypatch.setenv("DPSO_BOUND_PEEL", peel)
    rng = np.random.default_rng(int(rmax))
    for n in (40, 130, 400, 1000):
        cost = random_euclidean_matrix(n, rng)
        check(pkg, cost, perms(rng, 40, n), ("rmax", rmax, n))
        check(pkg, grid(n), perms(rng, 40, n), ("rmax-grid", rmax, n))


def test_bound_many_particles(pkg):
    rng = np.random.default_rng(43)
    for n, P in ((300, 12000), (500, 16384)):
        cost = grid(n) if n == 500 else np.floor(
            random_euclidean_matrix(n, rng) * 100.0)
        check(pkg, cost, perms(rng, P, n), ("many", n, P), 64, rng)


def test_bound_fallback_count(pkg, monkeypatch):
    # the context reports how many particles the bounded scan handed to the
    # band scan in its last pass; a small row list sends many there, and
    # the solve still follows the oracle
    from paper_1706_04399_b200.solver import numpy_stream_states
    rng = np.random.default_rng(19)
    n = 300
    cost = random_euclidean_matrix(n, rng)
    params = dict(n_particles=64, max_generations=8, stall_generations=8,
                  random_state=2)
    monkeypatch.setenv("DPSO_BOUND_PEEL", "0")
    for rmax, some in (("256", False), ("32", True)):
        monkeypatch.setenv("DPSO_BOUND_RMAX", rmax)
        s = pkg.DiscreteSwarmSolver(**params)
        ctx = s._make_context(cost)
        try:
            assert int(ctx.lib.dpso_scan_bound(ctx.h)) == 1
            ctx.set_streams(numpy_stream_states(2, 64 + 2))
            ctx.init(None, 0)
            counts = []
            for _ in range(8):
                ctx.step(1)
                counts.append(int(ctx.lib.dpso_bound_fallbacks(ctx.h)))
        finally:
            ctx.close()
        assert (max(counts) > 0) == some, (rmax, counts)
        gpu = pkg.DiscreteSwarmSolver(**params).fit(cost)
        ref = O.OracleSolver(**params).fit(cost)
        assert gpu.best_tour_ == ref.best_tour_
        assert gpu.convergence_ == ref.convergence_


@pytest.mark.parametrize("rmax,peel", [("256", "64"), ("32", "0"),
                                       ("32", "4")])
def test_bound_whole_solves_match_oracle(pkg, rmax, peel, monkeypatch):
    monkeypatch.setenv("DPSO_BOUND_RMAX", rmax)
    monkeypatch.setenv("DPSO_BOUND_PEEL", peel)
    rng = np.random.default_rng(41)
    for n, P, kind in ((60, 20, "int"), (90, 16, "euclid"), (49, 24, "grid")):
        cost = grid(n) if kind == "grid" else random_euclidean_matrix(n, rng)
        if kind == "int":
            cost = np.floor(cost * 100.0)
        params = dict(n_particles=P, max_generations=30, stall_generations=30,
                      random_state=5)
        gpu = pkg.DiscreteSwarmSolver(**params).fit(cost)
        ref = O.OracleSolver(**params).fit(cost)
        assert gpu.best_tour_ == ref.best_tour_
        assert gpu.convergence_ == ref.convergence_
        assert gpu.n_generations_ == ref.n_generations_


def test_bound_fallback_filter_overflow(pkg, monkeypatch):
    # particles handed to the band scan (peel limit 0, small row list) on a
    # non-integer lattice: thousands of exactly tied deltas overflow the
    # FILTER candidate lists, and the apply re-scans those particles in
    # fp64 itself (no separate re-scan kernel in bounded-scan mode)
    monkeypatch.setenv("DPSO_BOUND_RMAX", "32")
    monkeypatch.setenv("DPSO_BOUND_PEEL", "0")
    rng = np.random.default_rng(13)
    for n in (144, 400):
        cost = grid(n) / 3.0
        check(pkg, cost, perms(rng, 12, n), ("lattice-fallback", n))
        params = dict(n_particles=16, max_generations=12,
                      stall_generations=12, random_state=4)
        gpu = pkg.DiscreteSwarmSolver(**params).fit(cost)
        ref = O.OracleSolver(**params).fit(cost)
        assert gpu.best_tour_ == ref.best_tour_
        assert gpu.convergence_ == ref.convergence_
