"""Device cost-matrix build vs the reference's build_graph (golden) and the
Dijkstra oracle."""
import numpy as np
import pytest

from conftest import GOLDEN
from oracle import graph_oracle as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def gg():
    return np.load(f"{GOLDEN}/golden_graph.npz")


def unpack(gg, name):
    dims = tuple(int(v) for v in gg[f"{name}__dims"])
    return np.unpackbits(gg[f"{name}__occ"])[:np.prod(dims)].reshape(
        dims).astype(bool)


@pytest.mark.parametrize("name", ["wall", "ablation", "sealed"])
def test_scene_matrices_bit_exact(pkg, gg, name):
    cost, virt, vcost = pkg.build_cost_matrix(
        unpack(gg, name), gg[f"{name}__vox"], gg[f"{name}__weights"])
    assert np.array_equal(cost, gg[f"{name}__cost"])
    assert np.array_equal(virt, gg[f"{name}__virtual"])
    assert vcost == gg[f"{name}__vcost"][0]


def test_random_grids_vs_reference_astar(pkg, gg):
    rows = gg["grid_pairs"]
    for seed in range(12):
        occ = np.unpackbits(gg[f"grid{seed}__occ"])[:4000].reshape(
            20, 20, 10).astype(bool)
        sub = rows[rows[:, 0] == seed]
        vox = [sub[0, 1:4]] + [r[4:7] for r in sub]
        w = sub[0, 7:10]
        # a goal may coincide with the source or be occupied-free only
        cost, virt, vcost = pkg.build_cost_matrix(occ, np.array(vox), w)
        integral = all(float(x).is_integer() for x in w)
        for k, r in enumerate(sub):
            want = r[10]
            got = vcost if virt[0, k + 1] else cost[0, k + 1]
            if not np.isfinite(want):
                assert virt[0, k + 1]
            elif integral:
                assert got == want, (seed, k)
            else:
                assert abs(got - want) <= 1e-12 * want, (seed, k)


def test_larger_grid_vs_oracle(pkg):
    rng = np.random.default_rng(3)
    occ = rng.random((40, 30, 12)) < 0.25
    free = np.argwhere(~occ)
    vox = free[rng.choice(len(free), size=24, replace=False)]
    for w in [(1.0, 1.0, 1.0), (2.0, 1.0, 3.0)]:
        cost, virt, vcost = pkg.build_cost_matrix(occ, vox, w)
        ocost, ovirt, ovc = G.build_cost(occ, vox, w)
        assert np.array_equal(cost, ocost)
        assert np.array_equal(virt, ovirt)
        assert vcost == ovc


def test_occupied_viewpoint_rejected(pkg):
    occ = np.zeros((5, 5, 5), dtype=bool)
    occ[2, 2, 2] = True
    with pytest.raises(ValueError, match="occupied"):
        pkg.build_cost_matrix(occ, [[0, 0, 0], [2, 2, 2]], (1, 1, 1))


def test_load_cost_matrix_device_and_fit(pkg, tmp_path):
    # graph.py:123-143 text format -> pinned host buffer -> device tensor
    # (the --matrix path, cli.py:219-220) -> fit on the device matrix
    from conftest import random_euclidean_matrix
    import torch
    rng = np.random.default_rng(9)
    for n in (1, 7, 60):
        c = random_euclidean_matrix(n, rng)
        path = tmp_path / f"m{n}.txt"
        pkg.save_cost_matrix(path, c)
        host = pkg.load_cost_matrix(path)
        dev, ld = pkg.load_cost_matrix_device(path)
        assert dev.is_cuda and ld >= n and ld % 8 == 0
        assert dev.shape == (n, ld)
        got = dev.cpu().numpy()
        assert np.array_equal(got[:, :n], host)
        assert not got[:, n:].any()
        if n > 3:
            params = dict(n_particles=16, max_generations=30,
                          stall_generations=30, random_state=4)
            a = pkg.DiscreteSwarmSolver(**params).fit(host)
            b = pkg.DiscreteSwarmSolver(**params).fit(dev)
            assert a.best_tour_ == b.best_tour_
            assert a.convergence_ == b.convergence_
            # an unpadded (n, n) device tensor is padded on the way in
            e = pkg.DiscreteSwarmSolver(**params).fit(
                torch.as_tensor(host, device="cuda"))
            assert e.best_tour_ == a.best_tour_
    with pytest.raises(ValueError, match="finite"):
        bad = torch.full((5, 8), float("inf"), dtype=torch.float64,
                         device="cuda")
        pkg.DiscreteSwarmSolver(n_particles=4).fit(bad)


def test_fit_on_explicit_device_keeps_current_device(pkg):
    # ADVICE: contexts run on their workspace's device; the caller's
    # current device is handed back (one-GPU box: cuda:0 both ways)
    import torch
    from conftest import random_euclidean_matrix
    c = random_euclidean_matrix(40, np.random.default_rng(3))
    before = torch.cuda.current_device()
    s = pkg.DiscreteSwarmSolver(n_particles=12, max_generations=10,
                                device="cuda:0", random_state=1).fit(c)
    assert torch.cuda.current_device() == before
    assert sorted(s.best_tour_[:-1]) == list(range(40))


def _sharded_build(pkg, occ, vox, w, world):
    """The sharded build's device steps on one GPU: every rank's
    dpso_build_cost_rows block, concatenated (what gather_rows returns),
    then dpso_build_cost_assemble."""
    import ctypes

    import torch
    from paper_1706_04399_b200 import _lib
    from paper_1706_04399_b200.graph import _grid_args, source_blocks
    o, v, wt = _grid_args(occ, vox, w)
    n = len(v)
    lib = _lib.load()
    docc = torch.from_numpy(o.ravel()).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    B, blocks = source_blocks(n, world)
    parts = []
    for lo, hi in blocks:
        blk = torch.full((B, n), -1.0, dtype=torch.float64, device="cuda")
        _lib.check(lib.dpso_build_cost_rows(
            docc.data_ptr(), *o.shape, wt.ctypes.data_as(ctypes.c_void_p),
            v.ctypes.data_as(ctypes.c_void_p), n, lo, hi, blk.data_ptr(),
            stream))
        parts.append(blk)
    rows = torch.cat(parts)[:n].contiguous()
    ld = (n + 7) // 8 * 8
    cost = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    virt = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    vc = ctypes.c_double()
    _lib.check(lib.dpso_build_cost_assemble(
        rows.data_ptr(), n, cost.data_ptr(), ld, virt.data_ptr(),
        ctypes.byref(vc), stream))
    return (cost[:, :n].cpu().numpy(), virt.cpu().numpy().astype(bool),
            vc.value, rows.cpu().numpy())


@pytest.mark.parametrize("name", ["wall", "ablation", "sealed"])
def test_sharded_build_bit_exact(pkg, gg, name):
    # sources sharded, row blocks gathered, then assembled:
    # the reference's matrix for every shard count
    occ, vox, w = unpack(gg, name), gg[f"{name}__vox"], gg[f"{name}__weights"]
    for world in (2, 3, 8):
        cost, virt, vcost, rows = _sharded_build(pkg, occ, vox, w, world)
        assert np.array_equal(cost, gg[f"{name}__cost"]), world
        assert np.array_equal(virt, gg[f"{name}__virtual"]), world
        assert vcost == gg[f"{name}__vcost"][0]
        want = G.distance_rows(occ, vox, tuple(w), 0, len(vox))
        assert np.array_equal(rows, want)


def test_sharded_build_scene_scale(pkg):
    # the office scene (816 viewpoints): 8 shards == the one-call build
    import sys
    from conftest import ROOT
    sys.path.insert(0, f"{ROOT}/tools")
    import scenes
    occ, vox, w = scenes.scene("office")
    one = pkg.build_cost_matrix(occ, vox, w)
    cost, virt, vcost, _ = _sharded_build(pkg, occ, vox, w, 8)
    assert np.array_equal(cost, one[0])
    assert np.array_equal(virt, one[1])
    assert vcost == one[2]


def test_build_rows_errors(pkg, gg):
    import ctypes

    import torch
    from paper_1706_04399_b200 import _lib
    from paper_1706_04399_b200.graph import _grid_args
    occ, vox, w = _grid_args(unpack(gg, "wall"), gg["wall__vox"],
                             gg["wall__weights"])
    n = len(vox)
    lib = _lib.load()
    docc = torch.from_numpy(occ.ravel()).cuda()
    blk = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    args = (docc.data_ptr(), *occ.shape, w.ctypes.data_as(ctypes.c_void_p),
            vox.ctypes.data_as(ctypes.c_void_p), n)
    for lo, hi in ((-1, 2), (3, 2), (0, n + 1)):
        with pytest.raises(ValueError, match="source range"):
            _lib.check(lib.dpso_build_cost_rows(*args, lo, hi,
                                                blk.data_ptr(), None))
    # an occupied viewpoint fails on every shard, even one not owning it
    bad = vox.copy()
    bad[-1] = np.argwhere(occ)[0]
    with pytest.raises(ValueError, match="occupied"):
        _lib.check(lib.dpso_build_cost_rows(
            *args[:5], bad.ctypes.data_as(ctypes.c_void_p), n, 0, 1,
            blk.data_ptr(), None))


def test_build_cost_matrix_return_device(pkg, gg):
    occ, vox, w = unpack(gg, "wall"), gg["wall__vox"], gg["wall__weights"]
    cost, virt, vcost = pkg.build_cost_matrix(occ, vox, w,
                                              return_device=True)
    n = len(vox)
    assert cost.is_cuda and virt.is_cuda
    assert np.array_equal(cost[:, :n].cpu().numpy(), gg["wall__cost"])
    # the device matrix feeds fit() without a host round trip
    res = pkg.DiscreteSwarmSolver(n_particles=8, max_generations=5,
                                  random_state=1).fit(cost)
    assert sorted(res.best_tour_[:-1]) == list(range(n))
