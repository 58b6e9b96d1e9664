"""GPU parity pins for the exact shapes the benchmark runs.

* The 2-opt scan variant behind each bench config (C2: persistent warps,
  several tasks per particle; C3: one task per particle, the non-persistent
  launch; C4: two column ranges, persistent) against the oracle's
  ``_best_exchange`` (solver.py:88-106) on random subsets of the batch.
* The reference's own trajectory at the headline instance (bench ``c2``:
  ``random_euclidean_matrix(1000, default_rng(1000))``, P=1024), from
  fixtures made by running the unmodified reference
  (``tests/golden/make_golden_c2.py``).
* The reference's 12 golden ``_mutate`` swarms (solver.py:222-258, with
  duplicate, rotated and reflected tours) replayed through the device
  mutation pipeline (``dpso_mutate_step``).
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, random_euclidean_matrix
from oracle import dpso_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


def grid_matrix(n):
    """bench.py ``make_matrix`` for C3: L1 distances on a near-square grid."""
    side = int(math.ceil(math.sqrt(n)))
    idx = np.arange(n)
    pts = np.stack([idx % side, idx // side], 1).astype(float)
    return np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)


def random_tours(rng, P, n):
    return rng.permuted(np.tile(np.arange(n, dtype=np.int32), (P, 1)), axis=1)


def check_subset(pkg, cost, tours, rng, k, tag):
    new, delta = pkg.best_exchange_batch(cost, tours)
    pick = rng.choice(tours.shape[0], size=min(k, tours.shape[0]),
                      replace=False)
    for p in pick:
        eb, ed = O.best_exchange([int(v) for v in tours[p]], cost)
        assert new[p].tolist() == [int(v) for v in eb], (tag, int(p))
        assert float(delta[p]) == ed, (tag, int(p))
    # every row is still a permutation and the untouched rows kept delta 0
    assert (np.sort(new, axis=1) == np.arange(cost.shape[0])).all(), tag


def _lib():
    from paper_1706_04399_b200 import _lib as L
    return L.load()


@pytest.mark.parametrize("mode", [None, "column", "filter32",
                                  "exact32/rows32"])
def test_scan_one_task_per_particle_c3_shape(pkg, mode, monkeypatch):
    # C3: N=500 integer grid, P=16384.  Default: the band scan (EXACT, two
    # warp groups, ~110 particles per CTA); "column" and the modes: the
    # column scan, chunks == 1 -> the non-persistent
    # k_two_opt_scan32<16, EXACT32, fp16 rows> instantiation
    n, P = 500, 16384
    assert _lib().dpso_scan_chunks(n, P) == 1
    if mode == "column":
        monkeypatch.setenv("DPSO_SCAN_BAND", "0")
    elif mode:
        base, _, rows = mode.partition("/")
        monkeypatch.setenv("DPSO_SCAN_MODE", {"exact32": "1",
                                              "filter32": "2"}[base])
        if rows == "rows32":
            monkeypatch.setenv("DPSO_SCAN16", "0")
    rng = np.random.default_rng(500)
    cost = grid_matrix(n)
    tours = random_tours(rng, P, n)
    # a few rows that are 2-opt fixed points / near-optima (no move or tiny
    # moves) and exact duplicates
    nn, _ = O.nearest_neighbor_two_opt(cost)
    tours[:8] = np.array(nn[:-1], dtype=np.int32)
    tours[8:16] = tours[100]
    check_subset(pkg, cost, tours, rng, 256, ("c3", mode))
    new, delta = pkg.best_exchange_batch(cost, tours[:16])
    for p in range(16):
        eb, ed = O.best_exchange([int(v) for v in tours[p]], cost)
        assert new[p].tolist() == [int(v) for v in eb]
        assert float(delta[p]) == ed


@pytest.mark.parametrize("mode", [None, "exact32"])
def test_scan_nopersist_c3_integer_euclid(pkg, mode, monkeypatch):
    # the same one-task launch forced at a smaller batch on a wide-range
    # integer matrix (EXACT32 on fp32 rows when max|C| > 2048)
    monkeypatch.setenv("DPSO_SCAN_NOPERSIST", "1")
    if mode:
        monkeypatch.setenv("DPSO_SCAN_MODE", "1")
    rng = np.random.default_rng(77)
    for n in (33, 300, 640):
        cost = np.floor(random_euclidean_matrix(n, rng) * 1000.0)
        tours = random_tours(rng, 512, n)
        check_subset(pkg, cost, tours, rng, 64, ("nopersist", n, mode))


@pytest.mark.parametrize("scan", ["band", "column"])
def test_scan_c2_shape_persistent(pkg, scan, monkeypatch):
    # C2: N=1000 Euclidean, P=1024: the band scan (FILTER, two stages) by
    # default; the column scan (FILTER32, fp16 rows) has several tasks per
    # particle -> the persistent-warp launch
    if scan == "column":
        monkeypatch.setenv("DPSO_SCAN_BAND", "0")
    n, P = 1000, 1024
    assert _lib().dpso_scan_chunks(n, P) > 1
    rng = np.random.default_rng(1000)
    cost = random_euclidean_matrix(n, np.random.default_rng(1000))
    tours = random_tours(rng, P, n)
    check_subset(pkg, cost, tours, rng, 256, "c2")


def test_scan_c2_shape_nopersist(pkg, monkeypatch):
    monkeypatch.setenv("DPSO_SCAN_NOPERSIST", "1")
    n, P = 1000, 1024
    rng = np.random.default_rng(1001)
    cost = random_euclidean_matrix(n, np.random.default_rng(1000))
    tours = random_tours(rng, P, n)
    check_subset(pkg, cost, tours, rng, 128, "c2-nopersist")


def test_scan_c4_shape_two_column_ranges(pkg):
    # C4: N=2000 Euclidean, P=65536 -> two column ranges of 1024, two tasks
    # per particle, persistent warps
    n, P = 2000, 65536
    assert _lib().dpso_scan_chunks(n, P) == 2
    rng = np.random.default_rng(2000)
    cost = random_euclidean_matrix(n, np.random.default_rng(2000))
    tours = random_tours(rng, P, n)
    check_subset(pkg, cost, tours, rng, 256, "c4")


# --------------------------------------------------------------- C2 golden
def _golden_c2(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    with open(path) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["golden_c2_g8.json", "golden_c2_full.json"])
def test_c2_reference_trajectory(pkg, name):
    g = _golden_c2(name)
    cost = random_euclidean_matrix(1000, np.random.default_rng(1000))
    s = pkg.DiscreteSwarmSolver(**g["params"]).fit(cost)
    assert s.n_generations_ == g["n_generations"]
    assert s.convergence_ == g["convergence"]
    assert s.best_fitness_ == g["best_fitness"]
    assert list(s.best_tour_) == g["best_tour"]


# ------------------------------------------------------ golden _mutate swarms
def test_mutate_golden_swarms_on_device(pkg, golden_kernels):
    from paper_1706_04399_b200.solver import numpy_stream_states
    for r, rec in enumerate(golden_kernels["mutate"]):
        n, P = rec["n"], len(rec["before"])
        cost = np.array(rec["cost"], dtype=float)
        s = pkg.DiscreteSwarmSolver(n_particles=P, mutation_period=1,
                                    use_edge_exchange=False, random_state=0)
        ctx = s._make_context(cost)
        try:
            states = numpy_stream_states(0, P + 2)
            s0, inc, has, u = (int(v) for v in rec["rng_state"])
            m64 = (1 << 64) - 1
            states[1] = (s0 >> 64, s0 & m64, inc >> 64, inc & m64, has, u)
            ctx.set_streams(states)
            ctx.init(None, 0)  # prepares the first call's stream walk
            b = rec["before"]
            ctx.set_state(
                x=[p["body"] for p in b], pbest=[p["best_body"] for p in b],
                fit=[p["fitness"] for p in b],
                pfit=[p["best_fitness"] for p in b])
            ctx.mutate_step()
            st = ctx.state()
            for i, a in enumerate(rec["after"]):
                assert st["x"][i].tolist() == a["body"], (r, i)
                assert float(st["fit"][i]) == a["fitness"], (r, i)
                assert st["pbest"][i].tolist() == a["best_body"], (r, i)
                assert float(st["pfit"][i]) == a["best_fitness"], (r, i)
        finally:
            ctx.close()
