"""Pin the oracle restatement against golden vectors produced by running the
unmodified reference (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from conftest import golden_matrix, golden_params
from oracle import dpso_oracle as O
from oracle.np_random import PCG64Stream


def test_e2e_cases(golden_e2e):
    for case in golden_e2e["cases"]:
        cost = golden_matrix(golden_e2e, case["instance"])
        s = O.OracleSolver(**golden_params(golden_e2e, case)).fit(cost)
        assert list(s.best_tour_) == case["best_tour"], case["params"]
        assert s.best_fitness_ == case["best_fitness"]
        assert s.convergence_ == case["convergence"]
        assert s.n_generations_ == case["n_generations"]


def test_best_exchange(golden_kernels):
    for rec in golden_kernels["best_exchange"]:
        cost = golden_matrix(golden_kernels, rec["instance"])
        new, delta = O.best_exchange(rec["body"], cost)
        assert [int(v) for v in new] == rec["new_body"]
        assert delta == rec["delta"]
        assert O.tour_cost(rec["body"], cost.tolist()) == rec["cost"]


def test_mutate(golden_kernels):
    for rec in golden_kernels["mutate"]:
        n = rec["n"]
        P = len(rec["before"])
        st = O.SwarmState(n, P)
        for i, b in enumerate(rec["before"]):
            st.x[i] = list(b["body"])
            st.fit[i] = b["fitness"]
            st.pbest[i] = list(b["best_body"])
            st.pfit[i] = b["best_fitness"]
        s0, inc, h, u = rec["rng_state"]
        rng = PCG64Stream(s0, inc, h, u)
        O.OracleSolver(n_particles=P).mutate(st, rng, n, rec["cost"])
        for i, a in enumerate(rec["after"]):
            assert st.x[i] == a["body"]
            assert st.fit[i] == a["fitness"]
            assert st.pbest[i] == a["best_body"]
            assert st.pfit[i] == a["best_fitness"]


def test_nn_two_opt(golden_kernels):
    for rec in golden_kernels["nn_two_opt"]:
        cost = golden_matrix(golden_kernels, rec["instance"])
        tour, total = O.nearest_neighbor_two_opt(cost)
        assert list(tour) == rec["tour"]
        assert total == rec["cost"]


def test_canonical_and_operators(golden_kernels):
    for rec in golden_kernels["canonical"]:
        assert list(O.canonical_tour(rec["tour"])) == rec["canonical"]
    ops = golden_kernels["operators"]
    ex = ops["worked_example"]
    body = ex["x"][:-1]
    out = O.apply_open(body, [tuple(t) for t in ex["v"]])
    assert out + [out[0]] == ex["result"]
    for rec in ops["subtract"]:
        v = O.subtract_open(rec["x2"], rec["x1"])
        assert [list(t) for t in v] == rec["v"]
