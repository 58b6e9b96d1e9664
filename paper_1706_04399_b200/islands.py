"""Island model across GPUs: one swarm per rank, gbest
exchanged every K generations.

The swarm shards with no data-path collective; the only exchange is the
gbest migration:
  1. all_gather of a 16-byte record (gbest fitness fp64, rank) per island;
  2. every rank picks the winner: smallest fitness, lowest rank on ties;
  3. broadcast of the winner's tour (n int32) from the winning rank;
  4. each island adopts it iff strictly better than its own gbest
     (``dpso_offer_gbest``), so an island never gets worse.
Latency-bound (tens of microseconds over NVLink); amortised over K
generations.  Works with any torch.distributed backend (NCCL on the GPU box,
gloo in the CPU tests).

``exchange_device`` is the same exchange without a host round trip (NCCL):
each island packs (gbest fitness, rank, gbest tour) into a device record
(``dpso_island_pack``), one ``all_gather_into_tensor`` concatenates the
records of all ranks on the stream, and ``dpso_island_adopt`` picks the
winner and adopts it on the device - so generations keep streaming while
the exchange runs.
"""
from __future__ import annotations

import numpy as np


def pick_winner(records) -> tuple[int, float]:
    """records: iterable of (fitness, rank) -> (winner rank, fitness)."""
    best = None
    for fit, rank in records:
        key = (float(fit), int(rank))
        if best is None or key < best:
            best = key
    return best[1], best[0]


class IslandExchange:
    """``ctx`` needs ``result() -> (tour[n+1], fitness, conv)`` and
    ``offer_gbest(tour, fitness)`` (``solver.SwarmContext`` has both)."""

    def __init__(self, ctx, n: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.ctx, self.n, self.group = ctx, n, group
        backend = dist.get_backend(group)
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device())
                      if backend == "nccl" else torch.device("cpu"))
        self.device = device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.exchanges = 0
        self.adopted = 0

    def exchange(self) -> tuple[int, float]:
        torch, dist = self.torch, self.dist
        tour, fit, _ = self.ctx.result()
        rec = torch.tensor([fit, float(self.rank)], dtype=torch.float64,
                           device=self.device)
        recs = [torch.empty_like(rec) for _ in range(self.world)]
        dist.all_gather(recs, rec, group=self.group)
        winner, wfit = pick_winner((float(r[0]), int(r[1])) for r in recs)
        buf = torch.tensor(np.asarray(tour[:self.n], dtype=np.int32),
                           device=self.device)
        dist.broadcast(buf, src=dist.get_global_rank(self.group, winner)
                       if self.group is not None else winner,
                       group=self.group)
        self.exchanges += 1
        if winner != self.rank and wfit < fit:
            self.ctx.offer_gbest(buf.cpu().numpy(), wfit)
            self.adopted += 1
        return winner, wfit

    def exchange_device(self) -> None:
        """Stream-ordered exchange (needs ``ctx.island_pack/adopt`` and a
        backend whose tensors live on the GPU, i.e. NCCL)."""
        torch, dist = self.torch, self.dist
        if not hasattr(self, "_rec"):
            nbytes = self.ctx.island_record_bytes()
            self._rec = torch.empty(nbytes, dtype=torch.uint8,
                                    device=self.device)
            self._recs = torch.empty(nbytes * self.world, dtype=torch.uint8,
                                     device=self.device)
        self.ctx.island_pack(self._rec, self.rank)
        dist.all_gather_into_tensor(self._recs, self._rec, group=self.group)
        self.ctx.island_adopt(self._recs, self.world, self.rank)
        self.exchanges += 1
