"""The device bench harness (cli.py:178-274): every row's cost equals the
oracle's run of the same algorithm and seed (numpy-exact streams), with
several swarms in flight on separate CUDA streams; the CSV files keep the
reference's columns."""
import csv

import numpy as np
import pytest

from conftest import random_euclidean_matrix
from oracle import dpso_oracle as O


def _rows(path):
    with open(path) as fh:
        return list(csv.reader(fh))


def test_write_results_format(tmp_path):
    from paper_1706_04399_b200.bench_harness import BenchResult, write_results
    rows = [BenchResult("plain", "m", 0, 10.0, 0.5, 30),
            BenchResult("plain", "m", 1, 12.0, 0.7, 31),
            BenchResult("enhanced", "m", 0, 9.0, 0.25, 12),
            BenchResult("enhanced", "m", 1, 9.5, 0.75, 14)]
    write_results(tmp_path, rows, ["m"])
    res = _rows(tmp_path / "results.csv")
    assert res[0] == ["algorithm", "instance", "seed", "cost", "time",
                      "effort"]
    assert res[1] == ["plain", "m", "0", "10.0", "0.500000", "30"]
    summ = _rows(tmp_path / "summary.csv")
    assert summ[0] == ["instance", "algorithm", "mean_cost", "sd_cost",
                       "mean_time", "improvement_vs_plain_pct"]
    assert summ[1][:3] == ["m", "plain", "11.000000"]
    assert summ[2][1] == "enhanced" and summ[2][5] == "15.909"


@pytest.mark.gpu
def test_bench_matches_oracle(golden_e2e, tmp_path):
    from paper_1706_04399_b200.build import build
    build()
    from paper_1706_04399_b200.bench_harness import (ALGORITHMS, run_bench,
                                                    solver_params,
                                                    write_results)
    wall = np.array(golden_e2e["matrices"]["wall"], dtype=float)
    seed_tour = golden_e2e["seed_tours"]["wall"]
    euc = random_euclidean_matrix(40, np.random.default_rng(3))
    instances = [("wall", wall, seed_tour), ("euc40", euc, None)]
    base = solver_params(particles=24, generations=25, stall=10, seed=5)
    rows = run_bench(instances, trials=2, seed=5, base=base, workers=6)
    assert len(rows) == 2 * len(ALGORITHMS) * 2
    overrides = {
        "enhanced": lambda st: dict(seed_tour=st),
        "no_init": lambda st: dict(seed_tour=None, seed_fraction=0.0),
        "no_mutation": lambda st: dict(seed_tour=st, use_mutation=False),
        "no_edge_exchange": lambda st: dict(seed_tour=st,
                                            use_edge_exchange=False),
        "plain": lambda st: dict(seed_tour=None, seed_fraction=0.0,
                                 use_mutation=False, use_edge_exchange=False),
    }
    cost_of = {"wall": (wall, seed_tour), "euc40": (euc, None)}
    for r in rows:
        cost, st = cost_of[r.instance]
        if r.algorithm == "nn_2opt":
            assert r.cost == O.nearest_neighbor_two_opt(cost)[1]
            continue
        p = dict(base)
        p.update(random_state=r.seed, **overrides[r.algorithm](st))
        ref = O.OracleSolver(**p).fit(cost)
        assert r.cost == ref.best_fitness_, (r.instance, r.algorithm, r.seed)
        assert r.effort == ref.n_generations_
    write_results(tmp_path, rows, ["wall", "euc40"])
    assert len(_rows(tmp_path / "results.csv")) == len(rows) + 1
