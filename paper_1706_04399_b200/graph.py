"""Cost-matrix build on the device (replaces graph.py:41-78's pairwise A*).

``build_cost_matrix(occupancy, viewpoint_voxels, weights)`` returns
``(cost, virtual, virtual_cost)`` with the reference's semantics:
cost[i][j] = cost[j][i] = admissible-A* (= Dijkstra) motion cost on the
26-connected free-voxel graph (voxel.py:112-172), zero diagonal, blocked
pairs at ``1e3 * n * max_finite`` (1e6 when no finite edge) and flagged in
``virtual``.  ``build_graph(plan, grid, weights, heuristic_mode)`` is graph.py:41-78 for
callers holding the reference's CoveragePlan/VoxelGrid: the same
``TourGraph`` fields and ``leg(i, j)``, the same error for a viewpoint in
occupied space.  The waypoint legs are produced lazily: the reference's CLI
reads only the final tour's N legs (cli.py:122-133), so ``TourGraph.legs``
computes a pair's path on first access with a native restatement of the
reference's A* (same paths, byte for byte; ``tour_legs`` batches a tour's
legs over all host cores).  ``heuristic_mode="paper"`` (voxel.py:107-109:
the squared-distance priority, possibly suboptimal paths) takes every
pair's cost from that A* as the reference does; "admissible" costs come
from the device SSSP (equal to A*'s for a consistent heuristic).

``save_cost_matrix`` / ``load_cost_matrix`` are graph.py:123-143 (the
plain-text ``--matrix`` format) in native host code: the file bytes are the
reference's, and the reader parses straight into a pinned buffer that
``load_cost_matrix_device`` uploads without another copy.
"""
from __future__ import annotations

import ctypes
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InfeasibleViewpointError, OccupiedEndpointError
from .solver import _torch

VIRTUAL_SCALE = 1e3        # graph.py:17
_FALLBACK_VIRTUAL = 1e6    # graph.py:18


@dataclass(frozen=True)
class VoxelPath:
    """voxel.py:101-104."""
    waypoints: tuple
    motion_cost: float


class LazyLegs(Mapping):
    """graph.py's ``legs`` dict ((i, j), i < j -> VoxelPath; virtual pairs
    absent), with each path computed by the native A* on first access."""

    def __init__(self, occupancy, voxels, weights, mode, virtual):
        self._occ = occupancy
        self._vox = [tuple(int(c) for c in v) for v in voxels]
        self._w = tuple(float(x) for x in weights)
        self._mode = mode
        self._virtual = np.asarray(virtual, dtype=bool)
        self._cache = {}

    def _valid(self, key):
        i, j = key
        n = len(self._vox)
        return 0 <= i < j < n and not self._virtual[i, j]

    def prefetch(self, keys) -> None:
        """Compute the listed pairs in one native batch (all host cores)."""
        todo = [k for k in keys if self._valid(k) and k not in self._cache]
        if not todo:
            return
        pairs = [list(self._vox[i]) + list(self._vox[j]) for i, j in todo]
        for k, p in zip(todo, _voxel_paths(self._occ, pairs, self._w,
                                           self._mode)):
            self._cache[k] = None if p is None else VoxelPath(p[0], p[1])

    def __getitem__(self, key):
        key = (int(key[0]), int(key[1]))
        if not self._valid(key):
            raise KeyError(key)
        if key not in self._cache:
            self.prefetch([key])
        path = self._cache[key]
        if path is None:
            raise KeyError(key)
        return path

    def __iter__(self):
        n = len(self._vox)
        return ((i, j) for i in range(n) for j in range(i + 1, n)
                if not self._virtual[i, j])

    def __len__(self):
        n = len(self._vox)
        return int(np.triu(~self._virtual, 1).sum()) if n > 1 else 0


@dataclass(frozen=True)
class TourGraph:
    """graph.py:22-38."""
    n_nodes: int
    cost: np.ndarray
    virtual: np.ndarray
    virtual_cost: float
    legs: Mapping = field(default_factory=dict)

    def leg(self, i: int, j: int):
        """graph.py:30-38: the path from viewpoint i to j (reversed waypoints
        for i > j), None for i == j or a virtual edge."""
        if i == j:
            return None
        key = (i, j) if i < j else (j, i)
        path = self.legs.get(key)
        if path is not None and i > j:
            return VoxelPath(waypoints=tuple(reversed(path.waypoints)),
                             motion_cost=path.motion_cost)
        return path


def source_blocks(n: int, world: int):
    """The sharded build's source partition: rank r runs the
    SSSPs of sources [r*B, min(n, (r+1)*B)), B = ceil(n / world).  Every
    source costs one full-grid SSSP, so equal counts balance the ranks."""
    if n < 1 or world < 1:
        raise ValueError("n and world must be positive")
    B = -(-n // world)
    return B, [(min(n, r * B), min(n, (r + 1) * B)) for r in range(world)]


def gather_rows(block, n: int, group=None):
    """All-gather the ranks' (B, n) row blocks into the (n, n) table (one
    exchange step: NCCL over NVLink for device tensors, gloo on the host)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    full = torch.empty((world * block.shape[0], block.shape[1]),
                       dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(full, block.contiguous(), group=group)
    return full[:n]


def _grid_args(occupancy, viewpoint_voxels, weights):
    occ = np.ascontiguousarray(np.asarray(occupancy, dtype=bool),
                               dtype=np.uint8)
    if occ.ndim != 3:
        raise ValueError("occupancy must be a 3-D grid")
    vox = np.ascontiguousarray(np.asarray(viewpoint_voxels, dtype=np.int32)
                               .reshape(-1, 3))
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    return occ, vox, w


def build_cost_matrix(occupancy: np.ndarray, viewpoint_voxels, weights,
                      device=None, group=None, return_device=False):
    """graph.py:41-78's matrix from the device SSSP.  ``group``: a
    torch.distributed process group (one rank per GPU) to shard the sources
    over (``source_blocks``) and all-gather the row blocks; every rank gets
    the whole matrix, bit-identical to the single-GPU build.
    ``return_device``: (cost (n, ld) fp64, virtual (n, n) uint8) stay on
    the device, with the virtual cost."""
    torch = _torch()
    occ, vox, w = _grid_args(occupancy, viewpoint_voxels, weights)
    n = vox.shape[0]
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    lib = _lib.load()
    docc = torch.from_numpy(occ.ravel()).to(dev)
    ld = (n + 7) // 8 * 8
    cost = torch.zeros((n, ld), dtype=torch.float64, device=dev)
    virt = torch.zeros((n, n), dtype=torch.uint8, device=dev)
    vcost = ctypes.c_double(0.0)
    nx, ny, nz = occ.shape
    stream = torch.cuda.current_stream(dev).cuda_stream
    grid_args = (docc.data_ptr(), nx, ny, nz,
                 w.ctypes.data_as(ctypes.c_void_p),
                 vox.ctypes.data_as(ctypes.c_void_p), n)
    world = 1
    if group is not None:
        import torch.distributed as dist
        world = dist.get_world_size(group)
    if world == 1:
        _lib.check(lib.dpso_build_cost(*grid_args, cost.data_ptr(), ld,
                                       virt.data_ptr(), ctypes.byref(vcost),
                                       stream))
    else:
        import torch.distributed as dist
        B, blocks = source_blocks(n, world)
        lo, hi = blocks[dist.get_rank(group)]
        block = torch.zeros((B, n), dtype=torch.float64, device=dev)
        _lib.check(lib.dpso_build_cost_rows(*grid_args, lo, hi,
                                            block.data_ptr(), stream))
        rows = gather_rows(block, n, group)
        _lib.check(lib.dpso_build_cost_assemble(
            rows.data_ptr(), n, cost.data_ptr(), ld, virt.data_ptr(),
            ctypes.byref(vcost), stream))
    if return_device:
        return cost, virt, float(vcost.value)
    return (cost[:, :n].cpu().numpy(), virt.cpu().numpy().astype(bool),
            float(vcost.value))


def _paper_costs(occupancy, vox, weights):
    """Every pair's cost from the reference's A* with the paper heuristic
    (graph.py:58-66 with heuristic_mode="paper"), native, all host cores;
    blocked pairs virtual (graph.py:68-74).  Returns the paths too."""
    n = len(vox)
    keys = [(i, j) for i in range(n) for j in range(i + 1, n)]
    pairs = [list(vox[i]) + list(vox[j]) for i, j in keys]
    paths = _voxel_paths(occupancy, pairs, weights, "paper") if keys else []
    cost = np.zeros((n, n), dtype=float)
    virtual = np.zeros((n, n), dtype=bool)
    blocked = []
    for (i, j), p in zip(keys, paths):
        if p is None:
            blocked.append((i, j))
        else:
            cost[i, j] = cost[j, i] = p[1]
    max_finite = float(cost.max()) if n > 1 else 0.0
    vcost = (VIRTUAL_SCALE * n * max_finite if max_finite > 0
             else _FALLBACK_VIRTUAL)
    for i, j in blocked:
        cost[i, j] = cost[j, i] = vcost
        virtual[i, j] = virtual[j, i] = True
    return cost, virtual, vcost, dict(zip(keys, paths))


def build_graph(plan, grid, weights, heuristic_mode: str = "admissible"):
    """graph.py:41-78 (duck-typed plan.viewpoints / grid): the all-pairs
    obstacle-aware cost graph over the plan's viewpoints."""
    if heuristic_mode not in ("admissible", "paper"):
        raise ValueError(f"unknown heuristic_mode {heuristic_mode!r}")
    vox = []
    for vp in plan.viewpoints:
        idx = grid.point_to_voxel(vp.position)
        if not grid.is_free(idx):
            raise InfeasibleViewpointError(
                f"viewpoint {vp.id} maps to occupied voxel {idx}")
        vox.append(idx)
    occ = grid.occupancy
    if heuristic_mode == "paper":
        cost, virtual, vcost, paths = _paper_costs(occ, vox, weights)
    else:
        cost, virtual, vcost = build_cost_matrix(occ, vox, weights)
        paths = {}
    legs = LazyLegs(occ, vox, weights, heuristic_mode, virtual)
    for k, p in paths.items():
        legs._cache[k] = None if p is None else VoxelPath(p[0], p[1])
    cost.setflags(write=False)
    virtual.setflags(write=False)
    return TourGraph(n_nodes=len(vox), cost=cost, virtual=virtual,
                     virtual_cost=vcost, legs=legs)


def _path_bytes(path) -> bytes:
    import os
    return os.fsencode(os.fspath(path))


def save_cost_matrix(path, cost) -> None:
    """graph.py:123-130: header line n, then n lines of repr(float(x))."""
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise ValueError("cost matrix must be square")
    n = c.shape[0]
    with open(path, "w"):  # the reference's open() errors and truncation
        pass
    _lib.check(_lib.load().dpso_write_matrix_text(
        _path_bytes(path), c.ctypes.data_as(ctypes.c_void_p), n, n))


def _read_matrix(path, alloc):
    with open(path):  # the reference's open() errors (FileNotFoundError ...)
        pass
    lib = _lib.load()
    n = ctypes.c_int32(0)
    _lib.check(lib.dpso_read_matrix_text(_path_bytes(path), None, 0, 0,
                                         ctypes.byref(n)))
    buf, ptr, ld = alloc(int(n.value))
    _lib.check(lib.dpso_read_matrix_text(_path_bytes(path), ptr, ld,
                                         int(n.value), ctypes.byref(n)))
    return buf, int(n.value), ld


def load_cost_matrix(path) -> np.ndarray:
    """graph.py:133-143 (same values, same ValueError messages)."""
    def alloc(n):
        a = np.empty((n, n), dtype=np.float64)
        return a, a.ctypes.data_as(ctypes.c_void_p), n
    a, _, _ = _read_matrix(path, alloc)
    return a


def load_cost_matrix_device(path, device=None):
    """Parse into a pinned host buffer (rows padded to the device layout)
    and upload it: returns (cost tensor (n, ld) on the device, ld)."""
    torch = _torch()

    def alloc(n):
        ld = max(8, (n + 7) // 8 * 8)
        t = torch.zeros((max(n, 1), ld), dtype=torch.float64,
                        pin_memory=True)
        return t, ctypes.c_void_p(t.data_ptr()), ld
    host, n, ld = _read_matrix(path, alloc)
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    return host[:n].to(dev, non_blocking=False), ld


def _voxel_paths(occupancy, pairs, weights, heuristic_mode="admissible"):
    occ = np.ascontiguousarray(np.asarray(occupancy, dtype=bool),
                               dtype=np.uint8)
    if occ.ndim != 3:
        raise ValueError("occupancy must be a 3-D grid")
    if heuristic_mode not in ("admissible", "paper"):
        raise ValueError(f"unknown heuristic_mode {heuristic_mode!r}")
    pr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 6))
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    k = pr.shape[0]
    nx, ny, nz = occ.shape
    cap = nx * ny * nz  # a path visits each voxel at most once
    cap = min(cap, 1 << 16)
    while True:
        out = np.zeros((max(k, 1), cap, 3), dtype=np.int32)
        lens = np.zeros(max(k, 1), dtype=np.int64)
        costs = np.zeros(max(k, 1), dtype=np.float64)
        lib = _lib.load()
        rc = lib.dpso_voxel_paths(
            occ.ctypes.data_as(ctypes.c_void_p), nx, ny, nz,
            w.ctypes.data_as(ctypes.c_void_p),
            0 if heuristic_mode == "admissible" else 1,
            pr.ctypes.data_as(ctypes.c_void_p), k,
            out.ctypes.data_as(ctypes.c_void_p), cap,
            lens.ctypes.data_as(ctypes.c_void_p),
            costs.ctypes.data_as(ctypes.c_void_p))
        if rc != 0:
            msg = lib.dpso_last_error().decode()
            if "output capacity" in msg and cap < nx * ny * nz:
                cap = nx * ny * nz
                continue
            if "is occupied" in msg:
                raise OccupiedEndpointError(msg)
            _lib.check(rc)
        break
    res = []
    for i in range(k):
        if lens[i] == 0:
            res.append(None)
        else:
            res.append((tuple(tuple(int(v) for v in p)
                              for p in out[i, :lens[i]]), float(costs[i])))
    return res


def shortest_path(occupancy, start, goal, weights,
                  heuristic_mode="admissible"):
    """voxel.py:112-172: (waypoints, motion_cost), or None when blocked."""
    return _voxel_paths(occupancy, [list(start) + list(goal)], weights,
                        heuristic_mode)[0]


def tour_legs(occupancy, viewpoint_voxels, weights, tour,
              heuristic_mode="admissible") -> dict:
    """The legs of a closed tour as graph.py stores them: key (i, j) with
    i < j -> (waypoints from viewpoint i to j, motion cost); None for a
    blocked (virtual) edge.  TourGraph.leg(a, b) reverses for a > b."""
    vox = np.asarray(viewpoint_voxels, dtype=np.int32).reshape(-1, 3)
    keys = sorted({(min(a, b), max(a, b)) for a, b in zip(tour[:-1], tour[1:])
                   if a != b})
    pairs = [list(vox[i]) + list(vox[j]) for i, j in keys]
    paths = _voxel_paths(occupancy, pairs, weights, heuristic_mode)
    return dict(zip(keys, paths))
