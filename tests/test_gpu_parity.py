"""GPU parity: the CUDA path through the C ABI against the golden vectors of
the reference and against the oracle, bit for bit (permutations, argmin
choices, fitness bits — numpy-exact RNG streams make whole runs identical)."""
import numpy as np
import pytest

from conftest import golden_matrix, golden_params, random_euclidean_matrix
from oracle import dpso_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


def test_e2e_golden_runs(pkg, golden_e2e, scan_mode):
    for case in golden_e2e["cases"]:
        cost = golden_matrix(golden_e2e, case["instance"])
        s = pkg.DiscreteSwarmSolver(**golden_params(golden_e2e, case)).fit(cost)
        ctx = (case["instance"], case["params"])
        assert list(s.best_tour_) == case["best_tour"], ctx
        assert s.best_fitness_ == case["best_fitness"], ctx
        assert s.convergence_ == case["convergence"], ctx
        assert s.n_generations_ == case["n_generations"], ctx


def test_best_exchange_golden(pkg, golden_kernels):
    by_inst = {}
    for rec in golden_kernels["best_exchange"]:
        by_inst.setdefault(rec["instance"], []).append(rec)
    for inst, recs in by_inst.items():
        cost = golden_matrix(golden_kernels, inst)
        tours = np.array([r["body"] for r in recs], dtype=np.int32)
        new, delta = pkg.best_exchange_batch(cost, tours)
        for r, nb, d in zip(recs, new, delta):
            assert [int(v) for v in nb] == r["new_body"], inst
            assert float(d) == r["delta"], inst
        costs = pkg.tour_cost_batch(cost, tours)
        assert [float(c) for c in costs] == [r["cost"] for r in recs]


SCAN_MODES = {"fp64": "0", "exact32": "1", "filter32": "2"}


def set_scan_mode(monkeypatch, mode):
    # None: the default plan (the row-per-lane band scan where it applies);
    # "band/filter": the band scan forced to FILTER on integer matrices;
    # "column": the column-per-lane scan's default plan (DPSO_SCAN_BAND=0);
    # "<mode>" the column scan in that mode, fp16 rows where the mode allows
    # them; "<mode>/rows32" forces its fp32 rows (DPSO_SCAN16=0)
    if not mode:
        return
    if mode == "band/filter":
        monkeypatch.setenv("DPSO_BAND_MODE", "2")
        return
    if mode == "column":
        monkeypatch.setenv("DPSO_SCAN_BAND", "0")
        return
    base, _, rows = mode.partition("/")
    if base:
        monkeypatch.setenv("DPSO_SCAN_MODE", SCAN_MODES[base])
    if rows == "rows32":
        monkeypatch.setenv("DPSO_SCAN16", "0")


@pytest.fixture(params=[None, "band/filter", "column", "/rows32", "fp64",
                        "filter32", "filter32/rows32"])
def scan_mode(request, monkeypatch):
    set_scan_mode(monkeypatch, request.param)
    return request.param


def check_batch(pkg, cost, tours, tag):
    new, delta = pkg.best_exchange_batch(cost, tours)
    for t, nb, d in zip(tours, new, delta):
        eb, ed = O.best_exchange([int(v) for v in t], cost)
        assert [int(v) for v in nb] == [int(v) for v in eb], tag
        assert float(d) == ed, tag


def test_best_exchange_vs_oracle_sizes(pkg, scan_mode):
    rng = np.random.default_rng(3)
    for n in (4, 5, 31, 32, 33, 64, 65, 127, 300, 513, 1000, 1500, 2049, 2500):
        cost = random_euclidean_matrix(n, rng)
        tours = np.array([rng.permutation(n) for _ in range(6)],
                         dtype=np.int32)
        check_batch(pkg, cost, tours, (n, scan_mode))


@pytest.mark.parametrize("mode", [None, "/rows32", "fp64", "exact32",
                                  "exact32/rows32", "filter32",
                                  "filter32/rows32"])
@pytest.mark.parametrize("scale", [1.0, 300.0])
def test_best_exchange_integer_ties(pkg, mode, scale, monkeypatch):
    # integer costs: many exact ties -> row-major first-index tie break
    # (max |C| ~ 14 -> exact fp16 rows; ~ 4200 -> fp32 rows for EXACT32)
    set_scan_mode(monkeypatch, mode)
    rng = np.random.default_rng(8)
    for n in (17, 65, 300, 513, 1100):
        cost = np.floor(random_euclidean_matrix(n, rng) * scale)
        tours = np.array([rng.permutation(n) for _ in range(5)],
                         dtype=np.int32)
        check_batch(pkg, cost, tours, (n, mode))


def test_best_exchange_near_ties_and_converged(pkg, scan_mode):
    rng = np.random.default_rng(11)
    # a lattice with 1e-9 jitter: thousands of near-ties inside the fp32
    # filter window -> candidate-list overflow -> fp64 re-scan of the task
    side = 20
    g = np.stack(np.meshgrid(np.arange(side), np.arange(side)), -1)
    pts = g.reshape(-1, 2).astype(float) + rng.random((side * side, 2)) * 1e-9
    cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    tours = np.array([rng.permutation(side * side) for _ in range(4)] +
                     [np.arange(side * side)], dtype=np.int32)
    check_batch(pkg, cost, tours, ("lattice", scan_mode))
    # 2-opt-optimal tours: only the structural (i,i+1) residues are ~0
    for n in (50, 200):
        # (unscaled: at 1e4 the reference's own nearest_neighbor_two_opt
        # never terminates - no-op moves with fp64 residue < -1e-12 keep
        # firing, baselines.py:118-122)
        cost = random_euclidean_matrix(n, rng)
        tour, _ = O.nearest_neighbor_two_opt(cost)
        body = np.array([tour[:-1]], dtype=np.int32)
        check_batch(pkg, cost, body, ("converged", n, scan_mode))
    # a 2-opt-optimal tour across the fp32 scan's column ranges (n > 1024:
    # the structural pair (1023, 1024) sits on a range boundary), built by
    # the device NN + 2-opt (bit-exact to the oracle, test_nn_two_opt_golden)
    cost = random_euclidean_matrix(1100, rng)
    tour, _ = pkg.nearest_neighbor_two_opt(cost)
    body = np.array([list(tour)[:-1]], dtype=np.int32)
    check_batch(pkg, cost, body, ("converged", 1100, scan_mode))
    # large values: fp64 residues of the no-op pairs exceed 1e-12
    cost = random_euclidean_matrix(60, rng) * 1e9
    tours = np.array([rng.permutation(60) for _ in range(4)], dtype=np.int32)
    check_batch(pkg, cost, tours, ("big", scan_mode))


def test_best_exchange_fp16_rows_wide_range(pkg, scan_mode):
    # the fp16 filter's window scales with max |C|: a matrix with a few
    # huge entries (virtual edges, graph.py:63-78) and a tiny-valued one
    rng = np.random.default_rng(21)
    cost = random_euclidean_matrix(300, rng)
    blocked = rng.random(cost.shape) < 0.01
    blocked = blocked | blocked.T
    np.fill_diagonal(blocked, False)
    cost[blocked] = 1e3 * 300 * cost.max()
    tours = np.array([rng.permutation(300) for _ in range(4)], dtype=np.int32)
    check_batch(pkg, cost, tours, ("virtual", scan_mode))
    cost = random_euclidean_matrix(200, rng) * 1e-12
    tours = np.array([rng.permutation(200) for _ in range(4)], dtype=np.int32)
    check_batch(pkg, cost, tours, ("tiny", scan_mode))
    # asymmetric
    cost = random_euclidean_matrix(257, rng) * (1 + rng.random((257, 257)))
    np.fill_diagonal(cost, 0.0)
    tours = np.array([rng.permutation(257) for _ in range(4)], dtype=np.int32)
    check_batch(pkg, cost, tours, ("asym", scan_mode))


def test_scan_rows16_selected(pkg, monkeypatch):
    # the default plan streams fp16 rows for these matrices
    import ctypes
    from paper_1706_04399_b200.solver import device_cost
    rng = np.random.default_rng(5)
    for cost, want in ((random_euclidean_matrix(100, rng), 2),
                       (np.floor(random_euclidean_matrix(100, rng)), 1)):
        s = pkg.DiscreteSwarmSolver(n_particles=8)
        ctx = s._make_context(cost)
        try:
            assert ctx.lib.dpso_scan_mode(ctx.h) == want
            assert ctx.lib.dpso_scan_rows_bytes(ctx.h) == 2
        finally:
            ctx.close()


def test_nn_two_opt_golden(pkg, golden_kernels):
    for rec in golden_kernels["nn_two_opt"]:
        cost = golden_matrix(golden_kernels, rec["instance"])
        tour, total = pkg.nearest_neighbor_two_opt(cost)
        assert list(tour) == rec["tour"], rec["instance"]
        assert total == rec["cost"], rec["instance"]
        nn = pkg.nearest_neighbor_tour(cost)
        assert nn == O.nearest_neighbor_body(cost)


@pytest.mark.parametrize("n,P,G,kw", [
    # random_state 2923: the first mutation call's event 5 needs a Lemire
    # redraw (found by scanning seeds with oracle/np_random.py) -> exercises
    # the walk's redraw handling and the sampler's exact fallback
    (1000, 30, 3, {"mutation_period": 1, "use_edge_exchange": False,
                   "random_state": 2923}),
    (1000, 30, 2, {"mutation_period": 1, "random_state": 6395}),
    # n = 3000: the stream-walk ring no longer fits shared memory
    (3000, 8, 3, {"mutation_period": 1, "use_edge_exchange": False}),
    (40, 30, 25, {}),
    (40, 30, 25, {"mutation_period": 1}),
    (97, 24, 12, {"inertia": 0.5}),
    (130, 40, 10, {"seed_fraction": 0.3}),
    (260, 33, 6, {}),
    (200, 64, 8, {"use_edge_exchange": False, "mutation_period": 2}),
])
def test_per_generation_state_matches_oracle(pkg, n, P, G, kw):
    from paper_1706_04399_b200.solver import numpy_stream_states
    cost = random_euclidean_matrix(n, np.random.default_rng(n))
    seed = list(range(n)) + [0]
    params = dict(n_particles=P, max_generations=G, stall_generations=G,
                  random_state=n + P, seed_tour=seed)
    params.update(kw)
    orc = O.OracleSolver(**params)
    trace = []
    orc.fit(cost, trace=trace)
    gpu = pkg.DiscreteSwarmSolver(**params)
    seed_body, n_seed = gpu._seed(n)
    ctx = gpu._make_context(cost)
    try:
        ctx.set_streams(numpy_stream_states(params["random_state"], P + 2))
        ctx.init(seed_body, n_seed)
        for step, (_, st, gbest, gfit) in enumerate(trace):
            if step > 0:
                ctx.step(1)
            g = ctx.state()
            assert g["x"].tolist() == st.x, step
            assert g["fit"].tolist() == st.fit, step
            assert g["pbest"].tolist() == st.pbest, step
            assert g["pfit"].tolist() == st.pfit, step
            if gpu.inertia == 1.0:
                assert g["vmap"].tolist() == st.vmap, step
            assert g["gbest"].tolist() == gbest, step
            assert g["gbest_fit"] == gfit, step
    finally:
        ctx.close()


def test_full_size_properties(pkg):
    # BASELINE config-2 size (N=1000, P=1024), a few generations: every tour
    # stays a permutation, fitness equals the recomputed tour cost, the
    # convergence trace is monotone.
    n, P = 1000, 1024
    cost = random_euclidean_matrix(n, np.random.default_rng(1000))
    s = pkg.DiscreteSwarmSolver(n_particles=P, max_generations=6,
                                stall_generations=6, random_state=0)
    seed_body, n_seed = s._seed(n)
    from paper_1706_04399_b200.solver import numpy_stream_states
    ctx = s._make_context(cost)
    try:
        ctx.set_streams(numpy_stream_states(0, P + 2))
        ctx.init(None, 0)
        ctx.step(6)
        st = ctx.state()
        assert (np.sort(st["x"], axis=1) == np.arange(n)).all()
        assert (np.sort(st["pbest"], axis=1) == np.arange(n)).all()
        rec = pkg.tour_cost_batch(cost, st["x"])
        assert np.allclose(rec, st["fit"], rtol=1e-9, atol=0)
        tour, fit, conv = ctx.result()
        assert all(b <= a for a, b in zip(conv, conv[1:]))
        assert fit == conv[-1]
    finally:
        ctx.close()


def test_tour_cost_batch_large_n(pkg):
    # no shared-memory staging: any n (the earlier version staged 4 rows of
    # 8n bytes per CTA and stopped near n = 7000)
    rng = np.random.default_rng(21)
    n = 9000
    pts = rng.random((n, 2)) * 10.0
    cost = np.abs(pts[:, None, 0] - pts[None, :, 0]) + np.abs(
        pts[:, None, 1] - pts[None, :, 1])
    tours = np.array([rng.permutation(n) for _ in range(3)], dtype=np.int32)
    got = pkg.tour_cost_batch(cost, tours)
    for t, g in zip(tours, got):
        assert float(g) == O.tour_cost(list(t), cost)


def test_n_beyond_update_kernel_shared_memory_is_rejected(pkg):
    import ctypes
    from paper_1706_04399_b200 import _lib
    s = pkg.DiscreteSwarmSolver(n_particles=8)
    nbytes = ctypes.c_size_t(0)
    # 10 bytes per node (n > 6000): 30000 nodes need 300 KB
    rc = _lib.load().dpso_workspace_size(ctypes.byref(s._params()), 30000,
                                         ctypes.byref(nbytes))
    assert rc != 0
    msg = _lib.load().dpso_last_error().decode()
    assert "shared memory" in msg and "max n" in msg


@pytest.mark.gpu
@pytest.mark.parametrize("n,P,frac,rs", [
    (2, 5, 0.0, 1), (3, 7, 0.5, 2), (15, 32, 0.1, 0), (64, 300, 0.0, 5),
    (257, 129, 0.2, 9), (1000, 1024, 0.0, 0), (1500, 3000, 0.05, 11),
    (2000, 96, 1.0, 4),
])
def test_parallel_init_walk_matches_serial(pkg, monkeypatch, n, P, frac, rs):
    # The parallel init walk (every start's permutation length + pointer
    # doubling) must find exactly the cursors of the serial scan, which the
    # oracle pins (test_per_generation_state_matches_oracle, step 0).
    from paper_1706_04399_b200.solver import numpy_stream_states
    cost = random_euclidean_matrix(n, np.random.default_rng(n))
    seed = list(range(n)) + [0]
    states = {}
    for path in ("parallel", "serial"):
        if path == "serial":
            monkeypatch.setenv("DPSO_INIT_SERIAL", "1")
        s = pkg.DiscreteSwarmSolver(n_particles=P, max_generations=1,
                                    random_state=rs, seed_tour=seed,
                                    seed_fraction=frac)
        seed_body, n_seed = s._seed(n)
        ctx = s._make_context(cost)
        try:
            ctx.set_streams(numpy_stream_states(rs, P + 2))
            ctx.init(seed_body, n_seed)
            used = ctx.lib.dpso_init_path(ctx.h)
            assert used == (1 if path == "parallel" else 0), (path, used)
            states[path] = ctx.state()
            ctx.step(1)  # one generation from each init
            states[path + "1"] = ctx.state()
        finally:
            ctx.close()
    for key in ("x", "fit", "pbest", "gbest"):
        assert np.array_equal(states["parallel"][key], states["serial"][key])
        assert np.array_equal(states["parallel1"][key],
                              states["serial1"][key])
    if P * n <= 300 * 64:
        orc = O.OracleSolver(n_particles=P, max_generations=1,
                             random_state=rs, seed_tour=seed,
                             seed_fraction=frac)
        trace = []
        orc.fit(cost, trace=trace)
        assert states["parallel"]["x"].tolist() == trace[0][1].x


@pytest.mark.gpu
def test_lowmem_update_large_n(pkg, monkeypatch):
    # the 10-byte-per-node update (default for n > 14000; forced here by
    # DPSO_UPD_LOWMEM at n = 6500: targets read through the cache, sigma
    # folded into vmap in global memory): the same swarm state as the
    # 16-byte kernel generation by generation, and the oracle's after one
    # generation
    from paper_1706_04399_b200.solver import numpy_stream_states
    n, P, G = 6500, 12, 4
    cost = random_euclidean_matrix(n, np.random.default_rng(65))
    params = dict(n_particles=P, max_generations=G, stall_generations=G,
                  random_state=3, mutation_period=2)
    states = {}
    for kind in ("low", "full"):
        if kind == "low":
            monkeypatch.setenv("DPSO_UPD_LOWMEM", "1")
        else:
            monkeypatch.delenv("DPSO_UPD_LOWMEM", raising=False)
        s = pkg.DiscreteSwarmSolver(**params)
        ctx = s._make_context(cost)
        try:
            ctx.set_streams(numpy_stream_states(3, P + 2))
            ctx.init(None, 0)
            seq = []
            for _ in range(G):
                ctx.step(1)
                seq.append(ctx.state())
            states[kind] = seq
        finally:
            ctx.close()
    for a, b in zip(states["low"], states["full"]):
        for key in ("x", "pbest", "fit", "pfit", "vmap", "gbest"):
            assert np.array_equal(a[key], b[key]), key
    orc = O.OracleSolver(**dict(params, max_generations=1,
                                stall_generations=1))
    trace = []
    orc.fit(cost, trace=trace)
    _, st, gbest, gfit = trace[1]
    assert states["low"][0]["x"].tolist() == st.x
    assert states["low"][0]["vmap"].tolist() == st.vmap
    assert states["low"][0]["fit"].tolist() == st.fit


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [None, "/rows32", "exact32", "fp64"])
def test_best_exchange_nonmetric_integer(pkg, mode, monkeypatch):
    # integer, asymmetric, far from metric (EXACT32 scan): no structure for
    # the scan to lean on; many tours so the row bands take every parity
    set_scan_mode(monkeypatch, mode)
    rng = np.random.default_rng(31)
    for n in (37, 130, 301, 700):
        cost = rng.integers(0, 1000, size=(n, n)).astype(float)
        cost[rng.random((n, n)) < 0.3] = 0.0
        np.fill_diagonal(cost, 0.0)
        tours = np.array([rng.permutation(n) for _ in range(48)],
                         dtype=np.int32)
        check_batch(pkg, cost, tours, ("nonmetric", n, mode))


@pytest.mark.gpu
def test_island_adopt_on_device(pkg):
    # dpso_island_pack / dpso_island_adopt without NCCL: records of two
    # "other ranks" written by hand; the winner (smallest fitness, lowest
    # rank on ties) is adopted iff it is another rank's and strictly better
    import torch
    from paper_1706_04399_b200.solver import numpy_stream_states
    n, P = 30, 16
    cost = random_euclidean_matrix(n, np.random.default_rng(4))
    s = pkg.DiscreteSwarmSolver(n_particles=P, max_generations=3,
                                stall_generations=3, random_state=1)
    ctx = s._make_context(cost)
    try:
        ctx.set_streams(numpy_stream_states(1, P + 2))
        ctx.init(None, 0)
        ctx.step(2)
        nb = ctx.island_record_bytes()
        assert nb == 16 + (2 * 32 + 15) // 16 * 16
        recs = torch.zeros(3 * nb, dtype=torch.uint8, device="cuda")
        ctx.island_pack(recs[nb:2 * nb], 1)  # this island is rank 1
        own = ctx.state()
        mine = recs[nb:2 * nb].cpu().numpy()
        assert mine[:8].view(np.float64)[0] == own["gbest_fit"]
        assert mine[8:16].view(np.int64)[0] == 1
        assert mine[16:16 + 2 * n].view(np.uint16).tolist() == \
            own["gbest"].tolist()
        other = np.random.default_rng(9).permutation(n)

        def put(r, fit, tour):
            b = np.zeros(nb, np.uint8)
            b[:8] = np.frombuffer(np.float64(fit).tobytes(), np.uint8)
            b[8:16] = np.frombuffer(np.int64(r).tobytes(), np.uint8)
            b[16:16 + 2 * n] = np.frombuffer(
                tour.astype(np.uint16).tobytes(), np.uint8)
            recs[r * nb:(r + 1) * nb] = torch.from_numpy(b).cuda()
        # rank 2 ties rank 0 below ours: rank 0 wins the tie and is adopted
        put(0, own["gbest_fit"] - 1.0, other)
        put(2, own["gbest_fit"] - 1.0, other[::-1].copy())
        ctx.island_adopt(recs, 3, 1)
        got = ctx.state()
        assert got["gbest_fit"] == own["gbest_fit"] - 1.0
        assert got["gbest"].tolist() == other.tolist()
        # nobody better now (our own record wins): nothing changes
        ctx.island_pack(recs[nb:2 * nb], 1)
        put(0, got["gbest_fit"] + 5.0, np.arange(n))
        put(2, got["gbest_fit"], np.arange(n))
        ctx.island_adopt(recs, 3, 1)
        assert ctx.state()["gbest"].tolist() == other.tolist()
        ctx.step(1)  # the swarm carries on from the adopted gbest
    finally:
        ctx.close()


@pytest.mark.gpu
def test_island_exchange_device_nccl_single_rank(pkg):
    # the stream-ordered exchange through a real NCCL group (one rank: the
    # box has one GPU); its own record wins, so nothing is adopted
    import socket
    import torch
    import torch.distributed as dist
    from paper_1706_04399_b200.islands import IslandExchange
    from paper_1706_04399_b200.solver import numpy_stream_states
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}",
                            rank=0, world_size=1)
    try:
        n, P = 40, 16
        cost = random_euclidean_matrix(n, np.random.default_rng(6))
        s = pkg.DiscreteSwarmSolver(n_particles=P, max_generations=4,
                                    stall_generations=4, random_state=2)
        ctx = s._make_context(cost)
        try:
            ctx.set_streams(numpy_stream_states(2, P + 2))
            ctx.init(None, 0)
            ctx.step(2)
            before = ctx.state()
            ex = IslandExchange(ctx, n)
            ex.exchange_device()
            ctx.step(1)
            torch.cuda.synchronize()
            assert ex.exchanges == 1
            assert ctx.state()["gbest_fit"] <= before["gbest_fit"]
        finally:
            ctx.close()
    finally:
        dist.destroy_process_group()



def _with_virtual(cost, rng, frac):
    n = cost.shape[0]
    blk = np.triu(rng.random((n, n)) < frac, 1)
    blk = blk | blk.T
    out = cost.copy()
    out[blk] = 1e3 * n * cost.max()  # graph.py:63-78
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [None, "/rows32", "exact32", "filter32"])
def test_best_exchange_virtual_level_capped(pkg, mode, monkeypatch):
    # blocked pairs at 1e3 * n * max_finite: the scan caps that level in its
    # fp32/fp16 rows (orders pairs alike) and the apply re-evaluates the
    # chosen pair in fp64 - bit-exact against the oracle, integer (EXACT32)
    # and Euclidean (FILTER32), including tours that use virtual edges
    set_scan_mode(monkeypatch, mode)
    rng = np.random.default_rng(77)
    for n, integer in ((60, True), (300, True), (300, False), (1100, False)):
        base = random_euclidean_matrix(n, rng)
        if integer:
            base = np.floor(base * 20)
        cost = _with_virtual(base, rng, 0.02)
        tours = np.array([rng.permutation(n) for _ in range(16)],
                         dtype=np.int32)
        check_batch(pkg, cost, tours, ("virtual", n, integer, mode))


@pytest.mark.gpu
def test_swarm_with_virtual_edges_matches_oracle(pkg):
    # whole solve on a matrix with blocked pairs: convergence and tour
    # bit-identical to the oracle (the fitness += delta uses the fp64
    # re-evaluated delta)
    rng = np.random.default_rng(5)
    for integer in (True, False):
        base = random_euclidean_matrix(120, rng)
        if integer:
            base = np.floor(base * 20)
        cost = _with_virtual(base, rng, 0.05)
        params = dict(n_particles=24, max_generations=15,
                      stall_generations=15, random_state=4)
        ref = O.OracleSolver(**params).fit(cost)
        got = pkg.DiscreteSwarmSolver(**params).fit(cost)
        assert list(got.best_tour_) == list(ref.best_tour_)
        assert got.convergence_ == ref.convergence_


@pytest.mark.gpu
def test_best_exchange_negative_and_mixed_costs(pkg, scan_mode):
    # the reference does not forbid negative costs: mixed signs, integer and
    # not, one large negative outlier (no capping then: -max|C| occurs)
    rng = np.random.default_rng(99)
    for n in (40, 333):
        c = rng.normal(size=(n, n)) * 5
        np.fill_diagonal(c, 0.0)
        tours = np.array([rng.permutation(n) for _ in range(12)],
                         dtype=np.int32)
        check_batch(pkg, c, tours, ("normal", n, scan_mode))
        ci = np.round(c)
        check_batch(pkg, ci, tours, ("normal-int", n, scan_mode))
        co = c.copy()
        co[1, 2] = -1e6
        check_batch(pkg, co, tours, ("outlier", n, scan_mode))
