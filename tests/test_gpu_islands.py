"""The public island API (``IslandSolver``) on the GPU.

Two processes with real swarm contexts, both on cuda:0, exchanging over the
gloo host path (the NCCL device path is the same protocol on the stream),
must give exactly the run of the local mode (both islands in one process)
with the same seeds, and every island's tour must be a valid tour of the
reported fitness."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import random_euclidean_matrix

pytestmark = pytest.mark.gpu

PARAMS = dict(n_particles=24, max_generations=40, stall_generations=40,
              random_state=11)


def _cost():
    return random_euclidean_matrix(60, np.random.default_rng(60))


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1706_04399_b200 import IslandSolver
    s = IslandSolver(exchange_every=5, **PARAMS).fit(_cost())
    q.put((rank, s.best_tour_, s.best_fitness_, s.convergence_,
           s.n_generations_, s.island_fitness_, s.exchanges_))
    dist.barrier()
    dist.destroy_process_group()


def test_island_solver_two_processes_match_local_mode():
    from paper_1706_04399_b200 import IslandSolver
    from oracle.dpso_oracle import tour_cost
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    local = IslandSolver(exchange_every=5, devices=["cuda:0", "cuda:0"],
                         **PARAMS).fit(_cost())
    for rank, tour, fit, conv, gens, ifit, nex in out:
        assert tour == local.best_tour_, rank
        assert fit == local.best_fitness_
        assert conv == local.convergence_
        assert gens == local.n_generations_
        assert ifit == local.island_fitness_
    cost = _cost()
    assert sorted(local.best_tour_[:-1]) == list(range(60))
    assert abs(tour_cost(list(local.best_tour_[:-1]), cost.tolist()) -
               local.best_fitness_) <= 1e-9 * local.best_fitness_
    # the islands never end worse than their best member's start, and the
    # convergence trace is monotone
    assert all(a >= b for a, b in zip(local.convergence_,
                                      local.convergence_[1:]))


def test_island_solver_single_island_is_a_swarm():
    from paper_1706_04399_b200 import DiscreteSwarmSolver, IslandSolver
    from paper_1706_04399_b200.islands import island_seed
    s = IslandSolver(exchange_every=7, devices=["cuda:0"], **PARAMS).fit(
        _cost())
    p = dict(PARAMS, random_state=island_seed(PARAMS["random_state"], 0))
    ref = DiscreteSwarmSolver(**p).fit(_cost())
    assert s.best_tour_ == ref.best_tour_
    assert s.best_fitness_ == ref.best_fitness_
    assert s.convergence_ == ref.convergence_


def test_island_solver_device_matrix():
    # a CUDA-tensor matrix (build_cost_matrix(..., return_device=True) or
    # load_cost_matrix_device) is used in place: same run as the host one
    import torch
    from paper_1706_04399_b200 import IslandSolver
    cost = _cost()
    host = IslandSolver(exchange_every=5, devices=["cuda:0", "cuda:0"],
                        **PARAMS).fit(cost)
    dev = torch.from_numpy(cost).cuda()
    s = IslandSolver(exchange_every=5, devices=["cuda:0", "cuda:0"],
                     **PARAMS).fit(dev)
    assert s.best_tour_ == host.best_tour_
    assert s.best_fitness_ == host.best_fitness_
    assert s.convergence_ == host.convergence_
    assert s.island_fitness_ == host.island_fitness_
