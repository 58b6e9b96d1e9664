"""Island gbest exchange over torch.distributed, world_size 2, gloo on CPU
(the GPU box runs the same code over NCCL)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_1706_04399_b200.islands import IslandExchange, pick_winner


def test_pick_winner_ties_go_to_lowest_rank():
    assert pick_winner([(3.0, 0), (2.0, 1), (2.0, 2)]) == (1, 2.0)
    assert pick_winner([(1.0, 3), (1.0, 0)]) == (0, 1.0)


class FakeCtx:
    def __init__(self, tour, fit):
        self.tour, self.fit = list(tour), fit
        self.offers = []

    def result(self):
        return np.array(self.tour + [self.tour[0]]), self.fit, None

    def offer_gbest(self, tour, fit):
        self.offers.append((list(tour), fit))
        if fit < self.fit:
            self.tour, self.fit = list(tour), fit


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 6
    rng = np.random.default_rng(rank)
    tour = [int(v) for v in rng.permutation(n)]
    fit = [5.0, 3.0][rank]
    ctx = FakeCtx(tour, fit)
    ex = IslandExchange(ctx, n)
    winner, wfit = ex.exchange()
    # second exchange: nobody improves, nobody adopts again
    w2, f2 = ex.exchange()
    q.put((rank, winner, wfit, ctx.tour, ctx.fit, len(ctx.offers), tour,
           w2, f2))
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_world2_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r = q.get(timeout=120)
        out[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # rank 1 (fitness 3.0) wins; rank 0 adopts its tour exactly once
    assert out[0][1] == 1 and out[0][2] == 3.0
    assert out[1][1] == 1
    assert out[0][3] == out[1][6] and out[0][4] == 3.0
    assert out[0][5] == 1 and out[1][5] == 0
    assert out[0][7] == 0 and out[0][8] == 3.0  # tie -> lowest rank
