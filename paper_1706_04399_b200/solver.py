"""Drop-in ``DiscreteSwarmSolver`` running the enhanced DPSO on a B200.

Mirrors the reference estimator (``inspectour/solver.py:109-356``): same
constructor parameters (stored verbatim, sklearn ``BaseEstimator``), same
validation and error messages in ``fit`` (solver.py:139-172), same fitted
attributes ``best_tour_``, ``best_fitness_``, ``convergence_``,
``n_generations_``, ``report_``, and ``solve_matrix``.  With the default
``rng="numpy"`` the device reproduces the reference's numpy PCG64 streams
exactly (``SeedSequence(random_state).spawn(P + 2)``, solver.py:278-282), so a
fit returns the reference's tour and convergence trace bit for bit.

Extra keyword-only knobs (explicit parameters, as sklearn requires):
``rng`` ("numpy" | "philox") and ``device`` (a CUDA device, default current).

All compute runs in ``libdpso.so`` (hand-written sm_100a CUDA); PyTorch only
provides device memory and the stream.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
from sklearn.base import BaseEstimator

from . import _lib


@dataclass
class SolveReport:
    """solver.py:23-30."""
    best_tour: tuple[int, ...]
    best_fitness: float
    convergence: list[float]
    generations_run: int
    wall_time: float
    augmentation_flags: dict[str, bool] = field(default_factory=dict)


_M64 = (1 << 64) - 1


# numpy's SeedSequence constants (numpy/random/bit_generator.pyx)
_INIT_A, _MULT_A = 0x43B0D7E5, 0x931E8875
_INIT_B, _MULT_B = 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715
_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M32 = 0xFFFFFFFF
_M128 = (1 << 128) - 1


def _int_words(x: int) -> list:
    """numpy's _int_to_uint32_array."""
    if x == 0:
        return [0]
    out = []
    while x > 0:
        out.append(x & _M32)
        x >>= 32
    return out


def _spawned_pcg64_states(entropy: int, count: int) -> np.ndarray:
    """``SeedSequence(entropy).spawn(count)`` then ``PCG64(child).state``,
    vectorised over the children: the hash constants of SeedSequence's
    hashmix advance identically for every child, so the pool mixing and
    generate_state run as uint32 array arithmetic."""
    u32 = np.uint32
    i = np.arange(count, dtype=np.uint64)
    if count > 0 and int(i[-1]) > _M32:
        raise ValueError("too many streams")
    run = _int_words(entropy)
    run += [0] * max(0, 4 - len(run))  # a spawn key pads run entropy to 4
    ent = [np.full(count, w, dtype=u32) for w in run] + [i.astype(u32)]
    hc = _INIT_A

    def hashmix(v):
        nonlocal hc
        v = v ^ u32(hc)
        hc = (hc * _MULT_A) & _M32
        v = v * u32(hc)
        return v ^ (v >> u32(16))

    def mix(x, y):
        r = u32(_MIX_L) * x - u32(_MIX_R) * y
        return r ^ (r >> u32(16))

    with np.errstate(over="ignore"):
        pool = [hashmix(ent[k]) for k in range(4)]
        for s in range(4):
            for t in range(4):
                if s != t:
                    pool[t] = mix(pool[t], hashmix(pool[s]))
        for s in range(4, len(ent)):
            for t in range(4):
                pool[t] = mix(pool[t], hashmix(ent[s]))
        # generate_state(4, uint64): 8 uint32 words, little-endian pairs
        hb = _INIT_B
        w32 = []
        for k in range(8):
            v = pool[k % 4] ^ u32(hb)
            hb = (hb * _MULT_B) & _M32
            v = v * u32(hb)
            w32.append(v ^ (v >> u32(16)))
    w64 = [w32[2 * j].astype(np.uint64) | (w32[2 * j + 1].astype(np.uint64)
                                           << np.uint64(32)) for j in range(4)]
    s0, s1, i0, i1 = (w.tolist() for w in w64)
    rows = []
    for c in range(count):  # pcg64_set_seed -> pcg_setseq_128_srandom_r
        seed = (s0[c] << 64) | s1[c]
        inc = (((i0[c] << 64) | i1[c]) << 1 | 1) & _M128
        st = (inc + seed) & _M128            # state 0, step, += seed ...
        st = (st * _PCG_MULT + inc) & _M128  # ... step
        rows.append((st >> 64, st & _M64, inc >> 64, inc & _M64, 0, 0))
    return np.array(rows, dtype=np.uint64).reshape(count, 6)


def numpy_stream_states(random_state, count: int) -> np.ndarray:
    """PCG64 states of ``SeedSequence(random_state).spawn(count)`` as the
    (count, 6) uint64 records ``dpso_set_streams`` expects (solver.py:278-282:
    the reference spawns its streams this way).  Integer seeds take the
    vectorised restatement above (pinned against numpy by
    tests/test_lib_abi.py); any other entropy goes through numpy itself."""
    if isinstance(random_state, (int, np.integer)) and not isinstance(
            random_state, bool) and int(random_state) >= 0:
        if count <= 0xFFFFFFFF:
            # native (libdpso host code, threaded); the restatement above is
            # the same arithmetic in numpy
            words = np.array(_int_words(int(random_state)), dtype=np.uint32)
            out = np.empty((count, 6), dtype=np.uint64)
            _lib.check(_lib.load().dpso_spawn_pcg64_states(
                words.ctypes.data_as(ctypes.c_void_p), len(words), count,
                out.ctypes.data_as(ctypes.c_void_p)))
            return out
        return _spawned_pcg64_states(int(random_state), count)
    seqs = np.random.SeedSequence(random_state).spawn(count)
    out = np.empty((count, 6), dtype=np.uint64)
    for i, s in enumerate(seqs):
        st = np.random.PCG64(s).state
        a, b = st["state"]["state"], st["state"]["inc"]
        out[i] = (a >> 64, a & _M64, b >> 64, b & _M64, st["has_uint32"],
                  st["uinteger"])
    return out


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1706_04399_b200 needs a CUDA (sm_100a) device; there is no "
            "CPU fallback")
    return torch


def device_cost(X: np.ndarray, device=None):
    """Upload an n x n fp64 matrix into a zero-padded (n, ld) device tensor
    with ld = round_up(n, 8) (16-B aligned rows for the bulk row copies)."""
    torch = _torch()
    n = X.shape[0]
    ld = (n + 7) // 8 * 8
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    buf = torch.zeros((n, ld), dtype=torch.float64, device=dev)
    X = np.ascontiguousarray(X, dtype=float)
    with torch.cuda.device(dev):
        # native upload: pinned double buffer filled by host threads
        _lib.check(_lib.load().dpso_upload_matrix(
            X.ctypes.data, n, n, n, buf.data_ptr(), ld,
            torch.cuda.current_stream(dev).cuda_stream))
    return buf, ld


class SwarmContext:
    """Owns one device swarm (workspace tensor + ``dpso_ctx``)."""

    def __init__(self, params: "_lib.DpsoParams", n: int, cost_tensor, ld,
                 device=None):
        torch = _torch()
        self.lib = _lib.load()
        self.torch = torch
        self.params = params
        self.n = n
        self.device = cost_tensor.device
        nbytes = ctypes.c_size_t(0)
        _lib.check(self.lib.dpso_workspace_size(ctypes.byref(params), n,
                                                ctypes.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value), dtype=torch.uint8,
                                     device=self.device)
        self.cost = cost_tensor
        stream = torch.cuda.current_stream(self.device).cuda_stream
        h = ctypes.c_void_p()
        _lib.check(self.lib.dpso_create(
            ctypes.byref(params), n, self.workspace.data_ptr(),
            int(nbytes.value), stream, ctypes.byref(h)))
        self.h = h
        _lib.check(self.lib.dpso_set_cost(h, cost_tensor.data_ptr(), ld))

    def set_streams(self, states: np.ndarray) -> None:
        states = np.ascontiguousarray(states, dtype=np.uint64)
        _lib.check(self.lib.dpso_set_streams(
            self.h, states.ctypes.data_as(ctypes.c_void_p)))

    def init(self, seed_body, n_seed: int) -> None:
        if seed_body is not None and n_seed > 0:
            arr = np.ascontiguousarray(seed_body, dtype=np.int32)
            ptr = arr.ctypes.data_as(ctypes.c_void_p)
        else:
            arr, ptr, n_seed = None, None, 0
        _lib.check(self.lib.dpso_init(self.h, ptr, int(n_seed)))

    def run(self) -> int:
        g = ctypes.c_int32(0)
        _lib.check(self.lib.dpso_run(self.h, ctypes.byref(g)))
        return int(g.value)

    def step(self, gens: int) -> None:
        _lib.check(self.lib.dpso_step(self.h, int(gens)))

    def step_timed(self, gens: int):
        """Per-phase device ms over `gens` generations (dpso_step_timed)."""
        ms = np.zeros(6, dtype=np.float64)
        cnt = ctypes.c_int32(0)
        _lib.check(self.lib.dpso_step_timed(
            self.h, int(gens), ms.ctypes.data_as(ctypes.c_void_p),
            ctypes.byref(cnt)))
        return ms, int(cnt.value)

    def ctl(self):
        out = np.zeros(6, dtype=np.int32)
        gf = ctypes.c_double(0.0)
        _lib.check(self.lib.dpso_ctl(self.h, out.ctypes.data_as(
            ctypes.c_void_p), ctypes.byref(gf)))
        keys = ("gen", "stall", "done", "gens_run", "two_opt_count",
                "n_events")
        d = {k: int(v) for k, v in zip(keys, out)}
        d["gbest_fit"] = float(gf.value)
        return d

    def result(self):
        n = self.n
        tour = np.empty(n + 1, dtype=np.int32)
        fit = ctypes.c_double(0.0)
        conv = np.empty(self.params.max_generations + 1, dtype=np.float64)
        nconv = ctypes.c_int32(0)
        _lib.check(self.lib.dpso_result(
            self.h, tour.ctypes.data_as(ctypes.c_void_p), ctypes.byref(fit),
            conv.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nconv)))
        return tour, float(fit.value), conv[:nconv.value]

    def state(self):
        P, n = self.params.n_particles, self.n
        x = np.empty((P, n), np.int32)
        pb = np.empty((P, n), np.int32)
        vm = np.empty((P, n), np.int32)
        fit = np.empty(P, np.float64)
        pfit = np.empty(P, np.float64)
        gb = np.empty(n, np.int32)
        gf = ctypes.c_double(0.0)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _lib.check(self.lib.dpso_get_state(self.h, ptr(x), ptr(pb), ptr(fit),
                                           ptr(pfit), ptr(vm), ptr(gb),
                                           ctypes.byref(gf)))
        return {"x": x, "pbest": pb, "fit": fit, "pfit": pfit, "vmap": vm,
                "gbest": gb, "gbest_fit": float(gf.value)}

    def set_state(self, x=None, pbest=None, fit=None, pfit=None, vmap=None,
                  gbest=None, gbest_fit: float = 0.0) -> None:
        """Overwrite swarm state (P x n int32 tours, P fp64 values); None
        leaves a buffer as it is (dpso_set_state)."""
        keep = []

        def ptr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p)
        _lib.check(self.lib.dpso_set_state(
            self.h, ptr(x, np.int32), ptr(pbest, np.int32),
            ptr(fit, np.float64), ptr(pfit, np.float64), ptr(vmap, np.int32),
            ptr(gbest, np.int32), float(gbest_fit)))

    def mutate_step(self) -> None:
        """One mutation call without the update (dpso_mutate_step)."""
        _lib.check(self.lib.dpso_mutate_step(self.h))

    def offer_gbest(self, tour, fitness: float) -> None:
        arr = np.ascontiguousarray(tour, dtype=np.int32)
        _lib.check(self.lib.dpso_offer_gbest(
            self.h, arr.ctypes.data_as(ctypes.c_void_p), float(fitness)))

    def island_record_bytes(self) -> int:
        return int(self.lib.dpso_island_record_bytes(self.n))

    def island_pack(self, dev_record, rank: int) -> None:
        _lib.check(self.lib.dpso_island_pack(self.h, dev_record.data_ptr(),
                                             int(rank)))

    def island_adopt(self, dev_records, world: int, rank: int) -> None:
        _lib.check(self.lib.dpso_island_adopt(
            self.h, dev_records.data_ptr(), int(world), int(rank)))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.dpso_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DiscreteSwarmSolver(BaseEstimator):
    """Discrete PSO tour optimizer over a cost matrix (GPU).

    Parameters are those of the reference (solver.py:118-135) plus ``rng``
    and ``device``.  ``fit(X)`` expects a square cost matrix and exposes
    ``best_tour_``, ``best_fitness_``, ``convergence_``, ``n_generations_``
    and ``report_`` afterwards.
    """

    def __init__(self, n_particles=100, inertia=1.0, cognitive=0.4,
                 social=0.4, max_generations=200, stall_generations=30,
                 mutation_period=3, seed_fraction=0.1, seed_tour=None,
                 use_mutation=True, use_edge_exchange=True, parallel=False,
                 random_state=None, rng="numpy", device=None):
        self.n_particles = n_particles
        self.inertia = inertia
        self.cognitive = cognitive
        self.social = social
        self.max_generations = max_generations
        self.stall_generations = stall_generations
        self.mutation_period = mutation_period
        self.seed_fraction = seed_fraction
        self.seed_tour = seed_tour
        self.use_mutation = use_mutation
        self.use_edge_exchange = use_edge_exchange
        self.parallel = parallel
        self.random_state = random_state
        self.rng = rng
        self.device = device

    # -- validation (solver.py:139-162) -------------------------------------
    def _check_params(self):
        if self.n_particles < 3:
            raise ValueError("n_particles must be >= 3")
        for name in ("inertia", "cognitive", "social"):
            v = getattr(self, name)
            if not 0.0 <= v <= 1.0:
                raise ValueError(f"{name} must be in [0, 1], got {v}")
        if self.max_generations < 1:
            raise ValueError("max_generations must be >= 1")
        if self.stall_generations < 1:
            raise ValueError("stall_generations must be >= 1")
        if self.mutation_period < 1:
            raise ValueError("mutation_period must be >= 1")
        if not 0.0 <= self.seed_fraction <= 1.0:
            raise ValueError("seed_fraction must be in [0, 1]")
        if self.rng not in _lib.RNG_MODES:
            raise ValueError(f"rng must be one of {sorted(_lib.RNG_MODES)}")

    @staticmethod
    def _check_cost(X, finite: bool = True) -> np.ndarray:
        X = np.asarray(X, dtype=float)
        if X.ndim != 2 or X.shape[0] != X.shape[1]:
            raise ValueError(f"cost matrix must be square, got {X.shape}")
        if finite and not np.isfinite(X).all():
            raise ValueError("cost matrix must be finite")
        return X

    def _upload_cost(self, X):
        """solver.py:155-162's checks for a host matrix, with the
        finiteness test run on the uploaded copy (one device pass instead
        of a host pass over n^2 entries: 87 ms at n = 10000): (tensor, ld)."""
        cost = self._check_cost(X, finite=False)
        t, ld = device_cost(cost, self.device)
        if not bool(_torch().isfinite(t).all()):
            raise ValueError("cost matrix must be finite")
        return t, ld

    def _philox_seed(self) -> int:
        """64-bit Philox key from random_state (SeedSequence entropy)."""
        w = np.random.SeedSequence(self.random_state).generate_state(
            2, np.uint32)
        return int(w[0]) | (int(w[1]) << 32)

    def _params(self) -> "_lib.DpsoParams":
        return _lib.DpsoParams(
            n_particles=int(self.n_particles), inertia=float(self.inertia),
            cognitive=float(self.cognitive), social=float(self.social),
            max_generations=int(self.max_generations),
            stall_generations=int(self.stall_generations),
            mutation_period=int(self.mutation_period),
            seed_fraction=float(self.seed_fraction),
            use_mutation=int(bool(self.use_mutation)),
            use_edge_exchange=int(bool(self.use_edge_exchange)),
            parallel=int(bool(self.parallel)),
            rng_mode=_lib.RNG_MODES[self.rng],
            philox_seed=self._philox_seed() if self.rng == "philox" else 0)

    def _seed(self, n):
        """solver.py:167-174."""
        if self.seed_tour is not None and self.seed_fraction > 0:
            seed_body = [int(v) for v in list(self.seed_tour[:-1])]
            if sorted(seed_body) != list(range(n)):
                raise ValueError("seed_tour is not a tour over the matrix")
            n_seed = min(self.n_particles,
                         int(self.seed_fraction * self.n_particles + 0.5))
            return seed_body, n_seed
        return None, 0

    # -- main entry (solver.py:262-335) -------------------------------------
    def fit(self, X, y=None):
        """X: a square host cost matrix (the reference's input), or a CUDA
        tensor holding one - (n, n), or (n, ld) rows padded to ld >= n as
        ``load_cost_matrix_device`` returns them - which is used in place
        (no host round trip)."""
        self._check_params()
        dev_cost = self._device_cost(X)
        if dev_cost is None:
            cost = self._check_cost(X, finite=False)
            if cost.shape[0] == 1:  # the trivial solve needs no device
                self._check_cost(cost)
                dev_cost = (cost, 1)
            else:
                dev_cost = self._upload_cost(cost)
        n = dev_cost[0].shape[0]
        t0 = time.perf_counter()
        flags = {
            "init": self.seed_tour is not None and self.seed_fraction > 0,
            "mutation": self.use_mutation,
            "edge_exchange": self.use_edge_exchange,
            "parallel": self.parallel,
        }
        if n == 1:
            self._finish((0, 0), 0.0, [0.0], 1, t0, flags)
            return self
        seed_body, n_seed = self._seed(n)
        ctx = SwarmContext(self._params(), n, *dev_cost)
        try:
            if self.rng == "numpy":
                ctx.set_streams(numpy_stream_states(self.random_state,
                                                    self.n_particles + 2))
            ctx.init(seed_body, n_seed)
            gens = ctx.run()
            tour, fit, conv = ctx.result()
        finally:
            ctx.close()
        self._finish(tuple(int(v) for v in tour), fit,
                     [float(c) for c in conv], gens, t0, flags)
        return self

    @staticmethod
    def _device_cost(X):
        """(tensor (n, ld) float64 contiguous on a CUDA device, ld) for a
        device matrix, None for anything else."""
        if type(X).__module__.split(".")[0] != "torch":
            return None
        torch = _torch()
        if not (isinstance(X, torch.Tensor) and X.is_cuda):
            return None
        if X.ndim != 2 or X.shape[0] > X.shape[1]:
            raise ValueError(f"cost matrix must be square, got "
                             f"{tuple(X.shape)}")
        n, ld = X.shape
        if X.dtype != torch.float64 or not X.is_contiguous() or \
                (ld & 1) or X.data_ptr() % 16:
            ld = (n + 7) // 8 * 8
            buf = torch.zeros((n, ld), dtype=torch.float64, device=X.device)
            buf[:, :n].copy_(X[:, :n])
            X = buf
        if not bool(torch.isfinite(X[:, :n]).all()):
            raise ValueError("cost matrix must be finite")
        return X, ld

    def _make_context(self, cost: np.ndarray) -> SwarmContext:
        cost_t, ld = device_cost(cost, self.device)
        return SwarmContext(self._params(), cost.shape[0], cost_t, ld)

    def _finish(self, tour, fitness, convergence, generations, t0, flags):
        self.best_tour_ = tuple(int(x) for x in tour)
        self.best_fitness_ = float(fitness)
        self.convergence_ = [float(c) for c in convergence]
        self.n_generations_ = generations
        self.report_ = SolveReport(
            best_tour=self.best_tour_,
            best_fitness=self.best_fitness_,
            convergence=self.convergence_,
            generations_run=generations,
            wall_time=time.perf_counter() - t0,
            augmentation_flags=flags,
        )


def solve_matrix(cost, **params) -> SolveReport:
    """One-shot convenience wrapper (solver.py:352-356)."""
    solver = DiscreteSwarmSolver(**params)
    solver.fit(cost)
    return solver.report_
