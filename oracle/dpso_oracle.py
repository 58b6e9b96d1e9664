"""CPU restatement of the reference's enhanced-DPSO solve path.

TEST INFRASTRUCTURE ONLY — this module is the checker, never the product.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import it.  The product
path (``paper_1706_04399_b200``) never imports anything under ``oracle/``.

Every function cites the reference lines it restates
(``/root/reference/pkg/src/inspectour/solver.py`` unless noted).  Parity of
this restatement with the reference itself is pinned by
``tests/test_oracle_golden.py`` against fixtures in ``tests/golden/`` that were
produced by importing the reference (``tests/golden/make_golden.py``).

State is kept as explicit arrays (``x``, ``pbest``, ``vmap``, ``vinv``,
``fit``, ``pfit``) so that GPU state can be compared after every phase.
"""
from __future__ import annotations

import math

import numpy as np

from .np_random import PCG64Stream


# --------------------------------------------------------------------------
# helpers (solver.py:48-106, graph.py:106-115)
# --------------------------------------------------------------------------

def tour_cost(body, cost_rows) -> float:
    """``_tour_cost`` (solver.py:48-54): closing edge first, sequential fp64."""
    total = 0.0
    prev = body[-1]
    for node in body:
        total += cost_rows[prev][node]
        prev = node
    return total


def subtract_open(target, cur):
    """``_subtract_open`` (solver.py:57-69): left-to-right repair."""
    cur = list(cur)
    pos = {node: i for i, node in enumerate(cur)}
    out = []
    for i, want in enumerate(target):
        have = cur[i]
        if have != want:
            j = pos[want]
            cur[i], cur[j] = want, have
            pos[have], pos[want] = j, i
            out.append((have, want))
    return out


def apply_open(body, transpositions):
    """``_apply_open`` (solver.py:72-79): value transpositions in order."""
    body = list(body)
    pos = {node: i for i, node in enumerate(body)}
    for a, b in transpositions:
        ia, ib = pos[a], pos[b]
        body[ia], body[ib] = b, a
        pos[a], pos[b] = ib, ia
    return body


def prefix_len(c: float, length: int) -> int:
    """``_prefix_len`` (solver.py:82-85): round-half-up truncation."""
    if c <= 0.0:
        return 0
    return min(length, int(c * length + 0.5))


def best_exchange(body, cost: np.ndarray):
    """``_best_exchange`` (solver.py:88-106): best 2-opt move, first argmin."""
    n = len(body)
    if n < 4:
        return body, 0.0
    arr = np.asarray(body)
    succ = np.roll(arr, -1)
    d = cost[arr, succ]
    delta = (cost[np.ix_(arr, arr)] + cost[np.ix_(succ, succ)]
             - d[:, None] - d[None, :])
    delta[np.tril_indices(n)] = np.inf
    k = int(np.argmin(delta))
    i, j = divmod(k, n)
    if delta[i, j] < -1e-12:
        new = list(body)
        new[i + 1:j + 1] = reversed(new[i + 1:j + 1])
        return new, float(delta[i, j])
    return body, 0.0


def _f32_up(x):
    """x (float64 array) rounded up to float32."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    low = f.astype(np.float64) < x
    return np.where(low, np.nextafter(f, np.float32(np.inf)), f)


def _f32_down(x):
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    high = f.astype(np.float64) > x
    return np.where(high, np.nextafter(f, np.float32(-np.inf)), f)


def bounded_exchange(body, cost: np.ndarray, seeds: int = 32):
    """The bounded 2-opt scan's formulation (k_two_opt_bound.cu), restated
    to check on the CPU that it returns ``best_exchange``'s result.  Test
    infrastructure, not the reference: delta(i, j) >= -(h_i + h_j) with
    h_k = d_k - min((r(a_k) + r(s_k)) / 2, (q(a_k) + q(s_k)) / 2), r / q the
    off-diagonal row / column minima; h rounded up to fp32, the threshold
    -Tq - 2^-40 max|C| rounded down; Tq from the pairs of the `seeds` rows
    of largest h.  Only pairs with h_i + h_j >= thr are evaluated, with the
    reference expression.  Returns (new_body, delta, evaluated_pairs)."""
    n = len(body)
    if n < 4:
        return body, 0.0, 0
    arr = np.asarray(body)
    succ = np.roll(arr, -1)
    d = cost[arr, succ]
    off = cost + np.diag(np.full(n, np.inf))
    r = _f32_down(off.min(1)).astype(np.float64)
    q = _f32_down(off.min(0)).astype(np.float64)
    f = _f32_down(0.5 * (r[arr] + r[succ])).astype(np.float64)
    g = _f32_down(0.5 * (q[arr] + q[succ])).astype(np.float64)
    h = _f32_up(_f32_up(d).astype(np.float64) - np.minimum(f, g))
    h = h.astype(np.float64)

    def delta_of(i, j):
        return ((cost[arr[i], arr[j]] + cost[succ[i], succ[j]]) - d[i]) - d[j]

    seed = np.sort(np.argsort(-h, kind="stable")[:min(seeds, n)])
    si, sj = np.triu_indices(len(seed), 1)
    t0 = delta_of(seed[si], seed[sj]).min() if len(si) else np.inf
    tq = min(t0, -1e-12)
    slack = np.ldexp(np.abs(cost).max(), -40)
    thr = _f32_down(np.array([-tq - slack]))[0].astype(np.float64)
    ii, jj = np.triu_indices(n, 1)
    keep = _f32_up(h[ii] + h[jj]) >= thr
    ii, jj = ii[keep], jj[keep]
    if len(ii) == 0:
        return body, 0.0, 0
    dv = delta_of(ii, jj)
    k = np.lexsort((jj, ii, dv))[0]
    i, j, best = int(ii[k]), int(jj[k]), float(dv[k])
    if best < -1e-12:
        new = list(body)
        new[i + 1:j + 1] = reversed(new[i + 1:j + 1])
        return new, best, len(ii)
    return body, 0.0, len(ii)


def canonical_tour(sequence) -> tuple[int, ...]:
    """``canonical_tour`` (graph.py:106-115)."""
    body = list(sequence[:-1])
    k = body.index(0)
    body = body[k:] + body[:k]
    if len(body) > 2 and body[-1] < body[1]:
        body = [body[0]] + body[:0:-1]
    return tuple(body + [0])


def nearest_neighbor_body(cost: np.ndarray) -> list[int]:
    """Greedy construction of ``nearest_neighbor_two_opt``
    (baselines.py:110-116): from node 0, ties to the smallest index."""
    n = cost.shape[0]
    rows = cost.tolist()
    unvisited = set(range(1, n))
    body = [0]
    while unvisited:
        cur = body[-1]
        nxt = min(unvisited, key=lambda j: (rows[cur][j], j))
        unvisited.remove(nxt)
        body.append(nxt)
    return body


def nearest_neighbor_two_opt(cost: np.ndarray):
    """``nearest_neighbor_two_opt`` (baselines.py:103-123)."""
    n = cost.shape[0]
    if n == 1:
        return (0, 0), 0.0
    rows = cost.tolist()
    body = nearest_neighbor_body(cost)
    total = sum(rows[a][b] for a, b in zip(body, body[1:] + body[:1]))
    while True:
        body, delta = best_exchange(body, cost)
        if delta == 0.0:
            break
        total += delta
    return tuple(body) + (0,), float(total)


# --------------------------------------------------------------------------
# the parallel formulation of the prefix repair used by the CUDA update kernel
# --------------------------------------------------------------------------

def sigma_prefix(x, target, c: float):
    """Value permutation of the first ``prefix_len(c, L)`` transpositions of
    ``subtract_open(target, x)``, computed with the data-parallel formulation
    the CUDA update kernel uses (DESIGN.md §"update"):

    * pi(i) = pos_x(target[i]); emitting positions are the non-maximal
      positions of every non-trivial pi-cycle, so L = n - #cycles;
    * t = the k-th emitting position; for q <= t, cur_t[q] = target[q]; for
      q > t, cur_t[q] = target[r] with r the first position > t on the
      backward pi-orbit of q;
    * sigma(x[q]) = cur_t[q].

    Returns (sigma as a list indexed by value, k, L).  Restates, not copies,
    solver.py:57-69 + 82-85; equality with the sequential definition is
    pinned by tests/test_oracle_repair.py.
    """
    n = len(x)
    posx = [0] * n
    for i, v in enumerate(x):
        posx[v] = i
    pi = [posx[target[i]] for i in range(n)]
    back = [0] * n
    for i in range(n):
        back[pi[i]] = i
    # cycle maxima by walking (the kernel uses pointer jumping)
    cmax = [-1] * n
    for s in range(n):
        if cmax[s] >= 0:
            continue
        cyc = [s]
        q = pi[s]
        while q != s:
            cyc.append(q)
            q = pi[q]
        m = max(cyc)
        for q in cyc:
            cmax[q] = m
    emitting = [cmax[p] != p for p in range(n)]
    L = sum(emitting)
    k = prefix_len(c, L)
    sigma = list(range(n))
    if k == 0:
        return sigma, k, L
    cnt = 0
    t = -1
    for p in range(n):
        if emitting[p]:
            cnt += 1
            if cnt == k:
                t = p
                break
    cur = [0] * n
    for q in range(n):
        if q <= t:
            cur[q] = target[q]
        else:
            r = back[q]
            while r <= t:
                r = back[r]
            cur[q] = target[r]
    for q in range(n):
        sigma[x[q]] = cur[q]
    return sigma, k, L


# --------------------------------------------------------------------------
# the solver (solver.py:109-356) on explicit state arrays
# --------------------------------------------------------------------------

class SwarmState:
    """Explicit-array swarm state mirroring ``_Particle`` (solver.py:33-45)."""

    def __init__(self, n: int, p: int):
        self.n = n
        self.p = p
        self.x = [[0] * n for _ in range(p)]
        self.pbest = [[0] * n for _ in range(p)]
        self.fit = [0.0] * p
        self.pfit = [0.0] * p
        self.vmap = [list(range(n)) for _ in range(p)]
        self.vinv = [list(range(n)) for _ in range(p)]
        self.vel = [[] for _ in range(p)]   # transposition lists (w < 1)

    def copy(self) -> "SwarmState":
        s = SwarmState.__new__(SwarmState)
        s.n, s.p = self.n, self.p
        s.x = [list(r) for r in self.x]
        s.pbest = [list(r) for r in self.pbest]
        s.fit = list(self.fit)
        s.pfit = list(self.pfit)
        s.vmap = [list(r) for r in self.vmap]
        s.vinv = [list(r) for r in self.vinv]
        s.vel = [list(r) for r in self.vel]
        return s


class OracleSolver:
    """Restatement of ``DiscreteSwarmSolver`` (solver.py:109-349)."""

    def __init__(self, n_particles=100, inertia=1.0, cognitive=0.4,
                 social=0.4, max_generations=200, stall_generations=30,
                 mutation_period=3, seed_fraction=0.1, seed_tour=None,
                 use_mutation=True, use_edge_exchange=True, parallel=False,
                 random_state=None):
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

    # solver.py:278-282
    def make_streams(self):
        seqs = np.random.SeedSequence(self.random_state).spawn(
            self.n_particles + 2)
        return [PCG64Stream.from_seed_sequence(s) for s in seqs]

    # solver.py:166-188
    def init_swarm(self, n, cost_rows, init_rng: PCG64Stream) -> SwarmState:
        P = self.n_particles
        st = SwarmState(n, P)
        n_seed = 0
        seed_body = None
        if self.seed_tour is not None and self.seed_fraction > 0:
            seed_body = list(self.seed_tour[:-1])
            if sorted(seed_body) != list(range(n)):
                raise ValueError("seed_tour is not a tour over the matrix")
            n_seed = min(P, int(self.seed_fraction * P + 0.5))
        for i in range(P):
            if i < n_seed:
                body = list(seed_body)
                if i > 0 and n > 1:
                    a, b = init_rng.choice_noreplace(n, 2)
                    body[a], body[b] = body[b], body[a]
            else:
                body = init_rng.permutation(n)
            body = [int(v) for v in body]
            st.x[i] = body
            st.pbest[i] = list(body)
            st.fit[i] = st.pfit[i] = tour_cost(body, cost_rows)
        return st

    # solver.py:190-220
    def update_particle(self, st: SwarmState, i, gbest, cost_rows,
                        rng: PCG64Stream):
        r1, r2 = rng.random2()
        x = st.x[i]
        t1 = subtract_open(st.pbest[i], x)
        t1 = t1[:prefix_len(self.cognitive * r1, len(t1))]
        t2 = subtract_open(gbest, x)
        t2 = t2[:prefix_len(self.social * r2, len(t2))]
        if self.inertia == 1.0:
            vmap, vinv = st.vmap[i], st.vinv[i]
            for a, b in t1 + t2:
                ia, ib = vinv[a], vinv[b]
                vmap[ia], vmap[ib] = b, a
                vinv[a], vinv[b] = ib, ia
            st.x[i] = [vmap[v] for v in x]
        else:
            kept = st.vel[i][:prefix_len(self.inertia, len(st.vel[i]))]
            st.vel[i] = kept + t1 + t2
            st.x[i] = apply_open(x, st.vel[i])
        st.fit[i] = tour_cost(st.x[i], cost_rows)
        if st.fit[i] < st.pfit[i]:
            st.pfit[i] = st.fit[i]
            st.pbest[i] = list(st.x[i])

    # solver.py:222-258
    def mutate(self, st: SwarmState, mut_rng: PCG64Stream, n, cost_rows):
        P = st.p
        order = sorted(range(P), key=lambda i: (st.fit[i], i))
        seen = set()
        survivors, dropped = [], []
        for i in order:
            key = canonical_tour(st.x[i] + [st.x[i][0]])
            if key in seen:
                dropped.append(i)
            else:
                seen.add(key)
                survivors.append(i)
        keep = set(survivors[:math.ceil(len(survivors) / 3)])
        for rank, i in enumerate(dropped):
            src = survivors[rank % len(survivors)]
            st.x[i] = list(st.x[src])
            st.fit[i] = st.fit[src]
        k_hi = max(2, n // 4)
        for i in range(P):
            if i in keep:
                continue
            k = mut_rng.integers(1, k_hi + 1)
            k = min(k, n // 2)
            if k < 1:
                continue
            idxs = mut_rng.choice_noreplace(n, 2 * k)
            body = st.x[i]
            for t in range(k):
                a, b = idxs[2 * t], idxs[2 * t + 1]
                body[a], body[b] = body[b], body[a]
            st.fit[i] = tour_cost(body, cost_rows)
            if st.fit[i] < st.pfit[i]:
                st.pfit[i] = st.fit[i]
                st.pbest[i] = list(body)

    # solver.py:309-317
    def two_opt_all(self, st: SwarmState, cost: np.ndarray):
        for i in range(st.p):
            new_body, delta = best_exchange(st.x[i], cost)
            if delta < 0.0:
                st.x[i] = new_body
                st.fit[i] += delta
                if st.fit[i] < st.pfit[i]:
                    st.pfit[i] = st.fit[i]
                    st.pbest[i] = list(st.x[i])

    @staticmethod
    def argmin_first(fit) -> int:
        best = 0
        for i in range(1, len(fit)):
            if fit[i] < fit[best]:
                best = i
        return best

    # solver.py:262-335, split so one generation can be stepped and timed
    def start(self, X):
        """fit() up to the generation loop (solver.py:263-289)."""
        cost = np.asarray(X, dtype=float)
        self._cost = cost
        self._n = n = cost.shape[0]
        self._rows = cost.tolist()
        streams = self.make_streams()
        self._init_rng, self._mut_rng = streams[0], streams[1]
        self._prng = streams[2:]
        self.state_ = st = self.init_swarm(n, self._rows, self._init_rng)
        b = self.argmin_first(st.fit)
        self._gbest = list(st.x[b])
        self._gfit = st.fit[b]
        self._conv = [self._gfit]
        self._stall = 0
        self._gens = 0
        return self

    def generation(self) -> bool:
        """One pass of the generation loop (solver.py:292-328); returns
        True when the stall break fires."""
        st, n = self.state_, self._n
        gen = self._gens = self._gens + 1
        snap = list(self._gbest)
        for i in range(st.p):
            self.update_particle(st, i, snap, self._rows, self._prng[i])
        if self.use_mutation and gen % self.mutation_period == 0:
            self.mutate(st, self._mut_rng, n, self._rows)
        c = self.argmin_first(st.fit)
        improved = st.fit[c] < self._gfit
        self.last_two_opt_ = False
        if not improved and self.use_edge_exchange:
            self.last_two_opt_ = True
            self.two_opt_all(st, self._cost)
            c = self.argmin_first(st.fit)
            improved = st.fit[c] < self._gfit
        if improved:
            self._gfit = st.fit[c]
            self._gbest = list(st.x[c])
            self._stall = 0
        else:
            self._stall += 1
        self._conv.append(self._gfit)
        return self._stall >= self.stall_generations

    def fit(self, X, trace=None):
        cost = np.asarray(X, dtype=float)
        n = cost.shape[0]
        if n == 1:
            self.best_tour_ = (0, 0)
            self.best_fitness_ = 0.0
            self.convergence_ = [0.0]
            self.n_generations_ = 1
            return self
        self.start(cost)
        if trace is not None:
            trace.append(("init", self.state_.copy(), list(self._gbest),
                          self._gfit))
        for _ in range(self.max_generations):
            stop = self.generation()
            if trace is not None:
                trace.append((self._gens, self.state_.copy(),
                              list(self._gbest), self._gfit))
            if stop:
                break
        g = self._gbest
        self.best_tour_ = tuple(int(v) for v in g) + (int(g[0]),)
        self.best_fitness_ = float(self._gfit)
        self.convergence_ = [float(v) for v in self._conv]
        self.n_generations_ = self._gens
        return self
