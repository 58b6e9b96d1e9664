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


def island_seed(random_state, island: int) -> int:
    """random_state of island k: SeedSequence([random_state, k]) (island 0
    of a one-island run is NOT the plain random_state: an island run is a
    different algorithm from the single swarm, so it gets its own
    streams)."""
    ss = np.random.SeedSequence([int(random_state), int(island)])
    return int(ss.generate_state(1, np.uint64)[0] >> np.uint64(1))


class IslandSolver:
    """Island-model drop-in for ``DiscreteSwarmSolver.fit``.

    One swarm (island) per GPU, each with the given solver parameters;
    every ``exchange_every`` generations the islands exchange their gbest:
    the lowest fitness wins (lowest island on ties) and every island adopts
    the winner iff it is strictly better than its own gbest.  The run ends
    when every island has stopped (stall break) or after max_generations.

    Launch modes:
      * distributed: ``torch.distributed`` is initialized (one process per
        GPU, ``torchrun``) -> one island per rank on the rank's current
        device; the exchange is stream-ordered over NCCL
        (``IslandExchange.exchange_device``), or the host path on other
        backends (gloo);
      * local: ``devices=["cuda:0", "cuda:1", ...]`` -> one island per
        listed device in this process, stepped concurrently from host
        threads, exchanged on the host.

    Island k draws from ``island_seed(random_state, k)``.  Fitted
    attributes as ``DiscreteSwarmSolver`` (``best_tour_``, ``best_fitness_``,
    ``convergence_`` = the best gbest over the islands after each
    generation, ``n_generations_``, ``report_``) plus ``islands_``,
    ``exchanges_`` and ``island_fitness_``.
    """

    def __init__(self, exchange_every: int = 10, devices=None, group=None,
                 **params):
        if exchange_every < 1:
            raise ValueError("exchange_every must be >= 1")
        self.exchange_every = int(exchange_every)
        self.devices = list(devices) if devices is not None else None
        self.group = group
        self.params = dict(params)

    # -- helpers -------------------------------------------------------
    def _solver(self, island: int, device, base_seed: int):
        from .solver import DiscreteSwarmSolver
        p = dict(self.params)
        p["random_state"] = island_seed(base_seed, island)
        p["device"] = device
        return DiscreteSwarmSolver(**p)

    @staticmethod
    def _start(solver, cost, dev_cost=None, device=None):
        from .solver import SwarmContext, numpy_stream_states
        if dev_cost is not None:
            # a device matrix: used in place on its own GPU, copied once to
            # an island on another one
            t, ld = dev_cost
            if t.device != device:
                t = t.to(device)
            n = t.shape[0]
            seed_body, n_seed = solver._seed(n)
            ctx = SwarmContext(solver._params(), n, t, ld)
        else:
            seed_body, n_seed = solver._seed(cost.shape[0])
            ctx = solver._make_context(cost)
        if solver.rng == "numpy":
            ctx.set_streams(numpy_stream_states(solver.random_state,
                                                solver.n_particles + 2))
        ctx.init(seed_body, n_seed)
        return ctx

    def fit(self, X, y=None):
        import time
        import torch
        import torch.distributed as dist
        from .solver import DiscreteSwarmSolver, SolveReport
        probe = DiscreteSwarmSolver(**self.params)
        probe._check_params()
        # a CUDA tensor (e.g. build_cost_matrix(..., return_device=True))
        # stays on the device, as DiscreteSwarmSolver.fit takes it
        dev_cost = probe._device_cost(X)
        if dev_cost is None:  # uploaded once, checked on the device
            dev_cost = probe._upload_cost(X)
        cost = None
        n = dev_cost[0].shape[0]
        t0 = time.perf_counter()
        G = int(probe.max_generations)
        distributed = self.devices is None and dist.is_available() and \
            dist.is_initialized()
        base = probe.random_state
        if distributed:
            rank = dist.get_rank(self.group)
            world = dist.get_world_size(self.group)
            if base is None:  # one shared draw for every rank
                t = torch.tensor([np.random.SeedSequence().entropy % (1 << 62)
                                  if rank == 0 else 0], dtype=torch.int64)
                if dist.get_backend(self.group) == "nccl":
                    t = t.cuda()
                dist.broadcast(t, dist.get_global_rank(self.group, 0)
                               if self.group is not None else 0,
                               group=self.group)
                base = int(t.item())
            islands = [(rank, torch.device("cuda",
                                           torch.cuda.current_device()))]
        else:
            devs = self.devices or ["cuda:%d" % torch.cuda.current_device()]
            world = len(devs)
            if base is None:
                base = int(np.random.SeedSequence().entropy % (1 << 62))
            islands = [(k, torch.device(d)) for k, d in enumerate(devs)]
        if n == 1:
            probe.fit(X)
            self._copy(probe, world, 0)
            return self
        ctxs = []
        try:
            for k, dev in islands:
                with torch.cuda.device(dev):
                    ctxs.append(self._start(self._solver(k, dev, base), cost,
                                            dev_cost, dev))
            ex = None
            if distributed:
                ex = IslandExchange(ctxs[0], n, group=self.group)
            done_gens, exchanges = 0, 0
            while done_gens < G:
                step = min(self.exchange_every, G - done_gens)
                self._step_all(ctxs, islands, step)
                done_gens += step
                if distributed:
                    if dist.get_backend(self.group) == "nccl":
                        ex.exchange_device()
                    else:
                        ex.exchange()
                    flag = torch.tensor([int(ctxs[0].ctl()["done"])],
                                        dtype=torch.int32,
                                        device=ex.device)
                    dist.all_reduce(flag, op=dist.ReduceOp.MIN,
                                    group=self.group)
                    all_done = bool(flag.item())
                else:
                    self._exchange_local(ctxs, n)
                    all_done = all(c.ctl()["done"] for c in ctxs)
                exchanges += 1
                if all_done:
                    break
            res = [c.result() for c in ctxs]
            gens = [c.ctl()["gens_run"] for c in ctxs]
        finally:
            for c in ctxs:
                c.close()
        if distributed:
            tour, fit, conv = res[0]
            winner_tour, fit_all, conv_all, gens_all = self._gather(
                tour, fit, conv, gens[0], G, n, rank, world)
        else:
            fit_all = [r[1] for r in res]
            w = min(range(world), key=lambda k: (fit_all[k], k))
            winner_tour = res[w][0]
            conv_all = [self._pad(r[2], G) for r in res]
            gens_all = gens
        w = min(range(world), key=lambda k: (fit_all[k], k))
        ngen = max(gens_all)
        conv = np.min(np.stack(conv_all), axis=0)[:ngen + 1]
        self.best_tour_ = tuple(int(v) for v in winner_tour)
        self.best_fitness_ = float(fit_all[w])
        self.convergence_ = [float(c) for c in conv]
        self.n_generations_ = int(ngen)
        self.islands_ = world
        self.exchanges_ = exchanges
        self.island_fitness_ = [float(f) for f in fit_all]
        self.report_ = SolveReport(
            best_tour=self.best_tour_, best_fitness=self.best_fitness_,
            convergence=self.convergence_, generations_run=self.n_generations_,
            wall_time=time.perf_counter() - t0,
            augmentation_flags={
                "init": probe.seed_tour is not None and probe.seed_fraction > 0,
                "mutation": probe.use_mutation,
                "edge_exchange": probe.use_edge_exchange,
                "parallel": probe.parallel, "islands": world})
        return self

    def _copy(self, s, world, exchanges):
        self.best_tour_, self.best_fitness_ = s.best_tour_, s.best_fitness_
        self.convergence_, self.n_generations_ = s.convergence_, \
            s.n_generations_
        self.report_, self.islands_, self.exchanges_ = s.report_, world, \
            exchanges
        self.island_fitness_ = [s.best_fitness_]

    @staticmethod
    def _pad(conv, G):
        c = np.asarray(conv, dtype=np.float64)
        out = np.full(G + 1, c[-1] if len(c) else np.inf)
        out[:len(c)] = c
        return out

    @staticmethod
    def _step_all(ctxs, islands, step):
        if len(ctxs) == 1:
            ctxs[0].step(step)
            return
        import threading
        import torch
        errs = []

        def run(ctx, dev):
            try:
                with torch.cuda.device(dev):
                    ctx.step(step)
            except Exception as e:  # surfaced below
                errs.append(e)
        th = [threading.Thread(target=run, args=(c, d))
              for c, (_, d) in zip(ctxs, islands)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]

    @staticmethod
    def _exchange_local(ctxs, n):
        res = [c.result() for c in ctxs]
        wk, (wtour, wfit) = min(
            ((k, (r[0], r[1])) for k, r in enumerate(res)),
            key=lambda kv: (kv[1][1], kv[0]))
        for k, c in enumerate(ctxs):
            if k != wk and wfit < res[k][1]:
                c.offer_gbest(np.asarray(wtour[:n]), wfit)

    def _gather(self, tour, fit, conv, gens, G, n, rank, world):
        import torch
        import torch.distributed as dist
        dev = (torch.device("cuda", torch.cuda.current_device())
               if dist.get_backend(self.group) == "nccl"
               else torch.device("cpu"))
        rec = torch.tensor(np.concatenate([[fit, float(gens)],
                                           self._pad(conv, G)]),
                           dtype=torch.float64, device=dev)
        recs = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(recs, rec, group=self.group)
        recs = [r.cpu().numpy() for r in recs]
        fit_all = [float(r[0]) for r in recs]
        gens_all = [int(r[1]) for r in recs]
        conv_all = [r[2:] for r in recs]
        w = min(range(world), key=lambda k: (fit_all[k], k))
        buf = torch.tensor(np.asarray(tour[:n + 1], dtype=np.int32),
                           device=dev)
        dist.broadcast(buf, dist.get_global_rank(self.group, w)
                       if self.group is not None else w, group=self.group)
        return buf.cpu().numpy(), fit_all, conv_all, gens_all
