"""Kernel-level entry points mirroring the reference's private helpers.

* ``tour_cost_batch``      — ``_tour_cost`` (solver.py:48-54)
* ``best_exchange_batch``  — ``_best_exchange`` (solver.py:88-106)
* ``nearest_neighbor_tour``— NN construction (baselines.py:110-116)
* ``nearest_neighbor_two_opt`` — baselines.py:103-123 on the device

All run through ``libdpso.so``; inputs are numpy arrays, moved to the device
with torch.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .solver import _torch, device_cost


def _stream(t):
    return t.cuda.current_stream().cuda_stream


def tour_cost_batch(cost: np.ndarray, tours) -> np.ndarray:
    torch = _torch()
    cost = np.asarray(cost, dtype=float)
    tours = np.ascontiguousarray(tours, dtype=np.int32)
    n = cost.shape[0]
    cdev, ld = device_cost(cost)
    tdev = torch.from_numpy(tours).to(cdev.device)
    out = torch.empty(tours.shape[0], dtype=torch.float64, device=cdev.device)
    _lib.check(_lib.load().dpso_tour_cost_batch(
        cdev.data_ptr(), ld, n, tdev.data_ptr(), tours.shape[0],
        out.data_ptr(), _stream(torch)))
    return out.cpu().numpy()


def best_exchange_batch(cost: np.ndarray, tours):
    """Returns (new_tours, deltas) like ``_best_exchange`` per row."""
    torch = _torch()
    cost = np.asarray(cost, dtype=float)
    tours = np.ascontiguousarray(tours, dtype=np.int32)
    n = cost.shape[0]
    cdev, ld = device_cost(cost)
    tdev = torch.from_numpy(tours.copy()).to(cdev.device)
    delta = torch.empty(tours.shape[0], dtype=torch.float64,
                        device=cdev.device)
    _lib.check(_lib.load().dpso_best_exchange_batch(
        cdev.data_ptr(), ld, n, tdev.data_ptr(), tours.shape[0],
        delta.data_ptr(), _stream(torch)))
    return tdev.cpu().numpy(), delta.cpu().numpy()


def nearest_neighbor_tour(cost: np.ndarray, start: int = 0) -> list[int]:
    torch = _torch()
    cost = np.asarray(cost, dtype=float)
    n = cost.shape[0]
    cdev, ld = device_cost(cost)
    out = np.empty(n, dtype=np.int32)
    _lib.check(_lib.load().dpso_nn_tour(
        cdev.data_ptr(), ld, n, start, out.ctypes.data_as(ctypes.c_void_p),
        _stream(torch)))
    return [int(v) for v in out]


def nearest_neighbor_two_opt(cost: np.ndarray):
    """baselines.py:103-123: returns (closed tour, cost)."""
    torch = _torch()
    cost = np.asarray(cost, dtype=float)
    n = cost.shape[0]
    cdev, ld = device_cost(cost)
    out = np.empty(n + 1, dtype=np.int32)
    total = ctypes.c_double(0.0)
    _lib.check(_lib.load().dpso_nn_two_opt(
        cdev.data_ptr(), ld, n, out.ctypes.data_as(ctypes.c_void_p),
        ctypes.byref(total), _stream(torch)))
    return tuple(int(v) for v in out), float(total.value)
