"""GPU parity of the row-per-lane band scan (k_two_opt_band.cu) against the
oracle's ``_best_exchange`` (solver.py:88-106): band boundaries, EXACT and
FILTER rows, the single-stage launch for large n, the FILTER overflow
re-scan, asymmetric / negative / virtual-edge matrices, and whole solves."""
import math

import numpy as np
import pytest

from conftest import random_euclidean_matrix
from oracle import dpso_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _full_band_scan(monkeypatch):
    # the bounded scan (k_two_opt_bound.cu, tests/test_gpu_bound.py) would
    # take almost every random tour before the band scan sees it
    monkeypatch.setenv("DPSO_BOUND", "0")


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


def band_kind(pkg, cost, staging=False):
    s = pkg.DiscreteSwarmSolver(n_particles=4)
    ctx = s._make_context(cost)
    try:
        if staging:
            return int(ctx.lib.dpso_band_staging(ctx.h))
        return int(ctx.lib.dpso_scan_band(ctx.h))
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


def test_band_selected(pkg, monkeypatch):
    rng = np.random.default_rng(1)
    assert band_kind(pkg, grid(100)) == 1
    assert band_kind(pkg, random_euclidean_matrix(100, rng)) == 2
    big = np.floor(random_euclidean_matrix(100, rng) * 1e6)  # > 32767: FILTER
    assert band_kind(pkg, big) == 2
    monkeypatch.setenv("DPSO_SCAN_BAND", "0")
    assert band_kind(pkg, grid(100)) == 0


@pytest.mark.parametrize("staging", ["gather4", "bulk"])
@pytest.mark.parametrize("mode", ["exact", "filter"])
def test_band_boundaries(pkg, mode, staging, monkeypatch):
    # band edges (31 pair rows), 8-column groups, warp column splits; rows
    # staged by TMA gather4 (n <= ~960, the default) or one bulk copy each
    if mode == "filter":
        monkeypatch.setenv("DPSO_BAND_MODE", "2")
    if staging == "bulk":
        monkeypatch.setenv("DPSO_BAND_G4", "0")
    assert band_kind(pkg, grid(100), staging=True) == (
        2 if staging == "gather4" else 1)
    rng = np.random.default_rng(31)
    for n in list(range(4, 70)) + [93, 94, 95, 124, 125, 155, 156, 257, 511]:
        cost = np.floor(random_euclidean_matrix(n, rng) * 100.0)
        check(pkg, cost, perms(rng, 6, n), (mode, n))


def test_band_exact_ties(pkg):
    # integer grids: many exactly tied deltas; the first row-major argmin
    rng = np.random.default_rng(7)
    for n in (16, 49, 100, 500):
        cost = grid(n)
        check(pkg, cost, perms(rng, 24, n), ("grid", n))
        # 2-opt-optimal tours: no improving pair
        nn, _ = O.nearest_neighbor_two_opt(cost)
        check(pkg, cost, np.array([nn[:-1]] * 2, dtype=np.int32), ("opt", n))


def test_band_filter_scales(pkg):
    rng = np.random.default_rng(11)
    for n, mul in ((200, 1.0), (200, 1e-6), (200, 1e9), (300, 3.7)):
        cost = random_euclidean_matrix(n, rng) * mul
        check(pkg, cost, perms(rng, 16, n), ("scale", n, mul))
    # integers above the int16 range go through FILTER
    cost = np.floor(random_euclidean_matrix(300, rng) * 1e7)
    check(pkg, cost, perms(rng, 16, 300), "wide-int")


def test_band_filter_overflow_rescan(pkg):
    # a non-integer lattice: thousands of exactly tied deltas at the
    # minimum overflow the candidate lists -> the fp64 re-scan
    rng = np.random.default_rng(13)
    n = 144
    cost = grid(n) / 3.0
    check(pkg, cost, perms(rng, 12, n), "lattice")


def test_band_asymmetric_negative_virtual(pkg):
    rng = np.random.default_rng(17)
    n = 257
    c = random_euclidean_matrix(n, rng) * (1 + rng.random((n, n)))
    np.fill_diagonal(c, 0.0)
    check(pkg, c, perms(rng, 8, n), "asym")
    ci = np.floor(c * 50.0)
    check(pkg, ci, perms(rng, 8, n), "asym-int")
    neg = rng.normal(size=(n, n))
    check(pkg, neg, perms(rng, 8, n), "normal")
    check(pkg, np.round(neg * 100.0), perms(rng, 8, n), "normal-int")
    # blocked pairs (graph.py:63-78): one virtual level far above the rest
    v = np.floor(random_euclidean_matrix(n, rng) * 100.0)
    mask = np.triu(rng.random((n, n)) < 0.02, 1)
    mask = mask | mask.T
    v[mask] = 1e3 * n * v[~mask].max()
    check(pkg, v, perms(rng, 8, n), "virtual-int")
    ve = random_euclidean_matrix(n, rng)
    ve[mask] = 1e3 * n * ve[~mask].max()
    check(pkg, ve, perms(rng, 8, n), "virtual")


def test_band_largest_n(pkg):
    # the largest n whose two int16 stages fit shared memory, int8 rows past
    # it (n <= 2548), the column scan past that
    rng = np.random.default_rng(29)
    for n, kind in ((1000, 2), (1402, 2), (1403, 2), (2000, 2), (2548, 2),
                    (2549, 0)):
        cost = random_euclidean_matrix(n, rng)
        assert band_kind(pkg, cost) == kind, n
        check(pkg, cost, perms(rng, 300, n), ("large", n), 4, rng)
    cost = np.floor(random_euclidean_matrix(1400, rng) * 1000.0)
    assert band_kind(pkg, cost) == 1
    check(pkg, cost, perms(rng, 300, 1400), ("large-int", 1400), 6, rng)


def test_band_more_particles_than_ctas(pkg):
    # several particles per CTA: the column arrays prefetched during the
    # previous particle's last band
    rng = np.random.default_rng(37)
    for n, P in ((40, 1000), (333, 700)):
        cost = np.floor(random_euclidean_matrix(n, rng) * 100.0)
        check(pkg, cost, perms(rng, P, n), ("multi", n, P), 64, rng)
        check(pkg, cost / 7.0, perms(rng, P, n), ("multi-f", n, P), 64, rng)


@pytest.mark.parametrize("mode", ["exact", "filter"])
def test_band_int8_rows(pkg, mode, monkeypatch):
    # int8 rows (the default for 1402 < n <= 2548), forced at small n:
    # EXACT for integer matrices with |C| <= 127, FILTER at scale 2^k <=
    # 127 / max|C| otherwise; band edges, the overflow re-scan
    monkeypatch.setenv("DPSO_BAND_ES", "1")
    if mode == "filter":
        monkeypatch.setenv("DPSO_BAND_MODE", "2")
    rng = np.random.default_rng(59)
    for n in (4, 5, 31, 32, 33, 62, 63, 64, 65, 100, 155, 257, 300):
        cost = np.floor(random_euclidean_matrix(n, rng) * 80.0)  # <= 113
        check(pkg, cost, perms(rng, 6, n), ("int8", mode, n))
    for n, mul in ((200, 1.0), (200, 1e-6), (200, 1e9), (300, 3.7)):
        cost = random_euclidean_matrix(n, rng) * mul
        check(pkg, cost, perms(rng, 12, n), ("int8-scale", mode, n, mul))
    check(pkg, grid(144) / 3.0, perms(rng, 12, 144), ("int8-lattice", mode))
    v = np.floor(random_euclidean_matrix(257, rng) * 100.0)
    mask = np.triu(rng.random((257, 257)) < 0.02, 1)
    mask = mask | mask.T
    v[mask] = 1e3 * 257 * v[~mask].max()
    check(pkg, v, perms(rng, 8, 257), ("int8-virtual", mode))


def test_band_int8_large_integer(pkg):
    # n = 2000 integer costs above the int8 range: FILTER int8 rows
    rng = np.random.default_rng(61)
    cost = np.floor(random_euclidean_matrix(2000, rng) * 1000.0)
    assert band_kind(pkg, cost) == 2
    check(pkg, cost, perms(rng, 200, 2000), "int8-large-int", 4, rng)


@pytest.mark.parametrize("rpl", ["2", "1"])
@pytest.mark.parametrize("mode", ["exact", "filter"])
def test_band_two_rows_per_lane(pkg, mode, rpl, monkeypatch):
    # 64-slot bands (lane l: pair rows i0 + l and i0 + 32 + l), the default
    # for 64 <= n <= ~600: 63-row band edges, the second set's triangle,
    # partial last bands; DPSO_BAND_RPL=1 the 32-slot bands at the same n
    if mode == "filter":
        monkeypatch.setenv("DPSO_BAND_MODE", "2")
    monkeypatch.setenv("DPSO_BAND_RPL", rpl)
    rng = np.random.default_rng(53)
    for n in (64, 65, 66, 95, 96, 97, 126, 127, 128, 129, 189, 190, 191,
              252, 253, 300, 441, 500, 580, 600):
        cost = np.floor(random_euclidean_matrix(n, rng) * 100.0)
        check(pkg, cost, perms(rng, 5, n), (mode, rpl, n))
    cost = grid(500)
    check(pkg, cost, perms(rng, 300, 500), (mode, rpl, "grid"), 24, rng)


def test_band_gather4_limit(pkg):
    # the largest n whose shifted lines fit one gather4 box (2048 bytes:
    # 2n + 124 <= 2048) and the first n past it (bulk copies); partial last
    # groups of 4 rows
    rng = np.random.default_rng(47)
    for n in (957, 958, 962, 963, 964, 965):
        cost = np.floor(random_euclidean_matrix(n, rng) * 100.0)
        assert band_kind(pkg, cost, staging=True) == (2 if n <= 962 else 1)
        check(pkg, cost, perms(rng, 40, n), ("g4-limit", n), 8, rng)


def test_band_many_particles_per_cta(pkg):
    # ~100 particles per CTA, two warp groups on alternate bands (n = 300,
    # 500: four stages), the column arrays of a particle arriving on their
    # own barrier
    rng = np.random.default_rng(43)
    for n, P in ((300, 12000), (500, 16384)):
        side = int(math.ceil(math.sqrt(n)))
        cost = grid(n) if n == 500 else np.floor(
            random_euclidean_matrix(n, rng) * 100.0)
        check(pkg, cost, perms(rng, P, n), ("many", n, P), 48, rng)


def test_band_whole_solves_match_oracle(pkg):
    rng = np.random.default_rng(41)
    for n, P, kind in ((60, 20, "int"), (90, 16, "euclid")):
        cost = random_euclidean_matrix(n, rng)
        if kind == "int":
            cost = np.floor(cost * 100.0)
        params = dict(n_particles=P, max_generations=25, stall_generations=25,
                      random_state=5)
        gpu = pkg.DiscreteSwarmSolver(**params).fit(cost)
        ref = O.OracleSolver(**params).fit(cost)
        assert gpu.best_tour_ == ref.best_tour_
        assert gpu.convergence_ == ref.convergence_
