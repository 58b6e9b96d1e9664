"""The sharded cost-matrix build's host side (shard the SSSP
sources over ranks, all-gather the row blocks): the source partition, the
row exchange over torch.distributed (gloo, world_size 2 and 3, on CPU; the
GPU box runs the same ``gather_rows`` over NCCL), and the oracle split at
the exchange step against the reference goldens."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import GOLDEN
from oracle import graph_oracle as G
from paper_1706_04399_b200.graph import gather_rows, source_blocks


def unpack(gg, name):
    dims = tuple(int(v) for v in gg[f"{name}__dims"])
    return np.unpackbits(gg[f"{name}__occ"])[:np.prod(dims)].reshape(
        dims).astype(bool)


@pytest.mark.parametrize("n,world", [(1, 1), (1, 4), (5, 2), (7, 3),
                                     (8, 8), (100, 3), (1000, 8)])
def test_source_blocks_cover_once(n, world):
    B, blocks = source_blocks(n, world)
    assert len(blocks) == world and B * world >= n
    owned = [i for lo, hi in blocks for i in range(lo, hi)]
    assert owned == list(range(n))
    assert max(hi - lo for lo, hi in blocks) == B


def test_source_blocks_rejects_bad():
    with pytest.raises(ValueError):
        source_blocks(0, 2)
    with pytest.raises(ValueError):
        source_blocks(5, 0)


@pytest.mark.parametrize("name", ["wall", "ablation", "sealed"])
def test_split_oracle_matches_reference(name):
    gg = np.load(f"{GOLDEN}/golden_graph.npz")
    occ, vox = unpack(gg, name), gg[f"{name}__vox"]
    w = tuple(gg[f"{name}__weights"])
    n = len(vox)
    rows = np.concatenate([G.distance_rows(occ, vox, w, lo, hi)
                           for lo, hi in source_blocks(n, 3)[1]])
    cost, virt, vcost = G.assemble(rows)
    assert np.array_equal(cost, gg[f"{name}__cost"])
    assert np.array_equal(virt, gg[f"{name}__virtual"])
    assert vcost == gg[f"{name}__vcost"][0]


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gg = np.load(f"{GOLDEN}/golden_graph.npz")
    occ, vox = unpack(gg, name), gg[f"{name}__vox"]
    w = tuple(gg[f"{name}__weights"])
    n = len(vox)
    B, blocks = source_blocks(n, world)
    lo, hi = blocks[rank]
    block = torch.zeros((B, n), dtype=torch.float64)
    block[:hi - lo] = torch.from_numpy(G.distance_rows(occ, vox, w, lo, hi))
    rows = gather_rows(block, n).numpy()
    cost, virt, vcost = G.assemble(rows)
    ok = (np.array_equal(cost, gg[f"{name}__cost"])
          and np.array_equal(virt, gg[f"{name}__virtual"])
          and vcost == gg[f"{name}__vcost"][0])
    q.put((rank, ok, rows.shape))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "wall"), (3, "sealed")])
def test_gather_rows_gloo(world, name):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = len(np.load(f"{GOLDEN}/golden_graph.npz")[f"{name}__vox"])
    assert [g[0] for g in got] == list(range(world))
    assert all(g[1] for g in got), got
    assert all(tuple(g[2]) == (n, n) for g in got)
