"""CPU restatement of the reference's cost-matrix build.

TEST INFRASTRUCTURE ONLY — the checker, never the product (see
oracle/dpso_oracle.py for the rules).

* ``step_costs``  — voxel.py:25-38 (26 offsets in the reference order,
                    cost a1*alpha^2 + a2*beta^2 + a3*gamma^2)
* ``dijkstra_all`` — single-source Dijkstra over the 26-connected free-voxel
                    graph; admissible A* (voxel.py:112-172) returns the same
                    costs (its heuristic is consistent; the reference
                    asserts it, test_acceptance.py:120-144).  Bit-equal for
                    integer weights (every reference scene/test); with
                    non-integer weights A* may keep a path whose fp sum is
                    an ulp above the fp minimum
* ``build_cost``   — graph.py:41-78: pairwise costs for i < j from source i,
                    symmetric fill, blocked pairs -> VIRTUAL_SCALE * n *
                    max_finite (1e6 when no finite edge)
* ``distance_rows`` / ``assemble`` — the same build split at the sharded
                    build's exchange step: one rank's source rows, then
                    graph.py:63-78 over the gathered table

* ``save_cost_matrix`` / ``load_cost_matrix`` — graph.py:123-143, the
                    plain-text matrix format (repr(float(x)) entries)

Pinned against golden_graph.npz (tests/golden/make_golden_graph.py, run on
the unmodified reference) by tests/test_oracle_graph.py.
"""
from __future__ import annotations

import heapq
import math

import numpy as np

NEIGHBOR_STEPS = tuple((a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1)
                       for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0))
VIRTUAL_SCALE = 1e3
FALLBACK_VIRTUAL = 1e6


def step_costs(weights):
    a1, a2, a3 = weights
    return [a1 * a * a + a2 * b * b + a3 * c * c for a, b, c in NEIGHBOR_STEPS]


def dijkstra_all(occ: np.ndarray, weights, src) -> dict:
    """Distances from src to every reachable free voxel (dict index->cost)."""
    nx, ny, nz = occ.shape
    sc = step_costs(weights)
    src = tuple(int(v) for v in src)
    dist = {src: 0.0}
    heap = [(0.0, src)]
    done = set()
    while heap:
        g, cur = heapq.heappop(heap)
        if cur in done:
            continue
        done.add(cur)
        cx, cy, cz = cur
        for (dx, dy, dz), c in zip(NEIGHBOR_STEPS, sc):
            x, y, z = cx + dx, cy + dy, cz + dz
            if not (0 <= x < nx and 0 <= y < ny and 0 <= z < nz):
                continue
            if occ[x, y, z]:
                continue
            ng = g + c
            if ng < dist.get((x, y, z), math.inf):
                dist[(x, y, z)] = ng
                heapq.heappush(heap, (ng, (x, y, z)))
    return dist


def build_cost(occ: np.ndarray, vox, weights):
    """(cost, virtual, virtual_cost) as graph.py:41-78 computes them."""
    n = len(vox)
    vox = [tuple(int(c) for c in v) for v in vox]
    cost = np.zeros((n, n))
    virtual = np.zeros((n, n), dtype=bool)
    blocked = []
    for i in range(n):
        d = dijkstra_all(occ, weights, vox[i])
        for j in range(i + 1, n):
            c = d.get(vox[j])
            if c is None:
                blocked.append((i, j))
            else:
                cost[i, j] = cost[j, i] = c
    max_finite = float(cost.max()) if n > 1 else 0.0
    vcost = (VIRTUAL_SCALE * n * max_finite if max_finite > 0
             else FALLBACK_VIRTUAL)
    for i, j in blocked:
        cost[i, j] = cost[j, i] = vcost
        virtual[i, j] = virtual[j, i] = True
    return cost, virtual, vcost


def distance_rows(occ: np.ndarray, vox, weights, lo: int, hi: int):
    """Rows lo..hi-1 of the pairwise distance table (inf when blocked): the
    sources a rank of the sharded build owns (graph.py:58-66's loop body)."""
    n = len(vox)
    vox = [tuple(int(c) for c in v) for v in vox]
    rows = np.full((hi - lo, n), math.inf)
    for i in range(lo, hi):
        d = dijkstra_all(occ, weights, vox[i])
        for j in range(n):
            c = d.get(vox[j])
            if c is not None:
                rows[i - lo, j] = c
    return rows


def assemble(rows: np.ndarray):
    """graph.py:63-78 over a complete distance table (upper triangle)."""
    n = rows.shape[0]
    up = np.triu(np.ones((n, n), dtype=bool), 1)
    blocked = up & ~np.isfinite(rows)
    fin = up & np.isfinite(rows)
    max_finite = float(rows[fin].max()) if fin.any() else 0.0
    vcost = (VIRTUAL_SCALE * n * max_finite if max_finite > 0
             else FALLBACK_VIRTUAL)
    cost = np.where(fin, rows, 0.0)
    cost[blocked] = vcost
    cost = cost + cost.T
    virtual = blocked | blocked.T
    return cost, virtual, vcost


def save_cost_matrix(path, cost) -> None:
    """graph.py:123-130."""
    n = cost.shape[0]
    with open(path, "w") as fh:
        fh.write(f"{n}\n")
        for row in cost:
            fh.write(" ".join(repr(float(x)) for x in row))
            fh.write("\n")


def load_cost_matrix(path) -> np.ndarray:
    """graph.py:133-143."""
    with open(path) as fh:
        tokens = fh.read().split()
    if not tokens:
        raise ValueError(f"empty cost matrix file {path}")
    n = int(tokens[0])
    vals = [float(t) for t in tokens[1:]]
    if len(vals) != n * n:
        raise ValueError(
            f"cost matrix {path}: expected {n * n} entries, got {len(vals)}")
    return np.asarray(vals, dtype=float).reshape(n, n)
