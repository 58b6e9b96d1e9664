"""ctypes binding of ``libdpso.so`` (the C ABI in ``include/dpso.h``).

The library is built in-tree (``paper_1706_04399_b200/build.py``).  There is
no CPU fallback: if the library or a CUDA device is missing, every entry point
raises, loudly.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdpso.so")

DPSO_OK, DPSO_EINVAL, DPSO_ECUDA, DPSO_ECOMM = 0, 1, 2, 3
RNG_MODES = {"numpy": 0, "philox": 1}


class DpsoParams(ctypes.Structure):
    _fields_ = [
        ("n_particles", ctypes.c_int32),
        ("inertia", ctypes.c_double),
        ("cognitive", ctypes.c_double),
        ("social", ctypes.c_double),
        ("max_generations", ctypes.c_int32),
        ("stall_generations", ctypes.c_int32),
        ("mutation_period", ctypes.c_int32),
        ("seed_fraction", ctypes.c_double),
        ("use_mutation", ctypes.c_int32),
        ("use_edge_exchange", ctypes.c_int32),
        ("parallel", ctypes.c_int32),
        ("rng_mode", ctypes.c_int32),
        ("philox_seed", ctypes.c_uint64),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SIG = {
    "dpso_workspace_size": (_I32, [ctypes.POINTER(DpsoParams), _I32,
                                   ctypes.POINTER(ctypes.c_size_t)]),
    "dpso_create": (_I32, [ctypes.POINTER(DpsoParams), _I32, _P,
                           ctypes.c_size_t, _P, ctypes.POINTER(_P)]),
    "dpso_set_cost": (_I32, [_P, _P, _I64]),
    "dpso_set_streams": (_I32, [_P, _P]),
    "dpso_init": (_I32, [_P, _P, _I32]),
    "dpso_run": (_I32, [_P, ctypes.POINTER(_I32)]),
    "dpso_step": (_I32, [_P, _I32]),
    "dpso_scan_mode": (_I32, [_P]),
    "dpso_init_path": (_I32, [_P]),
    "dpso_scan_rows_bytes": (_I32, [_P]),
    "dpso_scan_band": (_I32, [_P]),
    "dpso_band_staging": (_I32, [_P]),
    "dpso_scan_bound": (_I32, [_P]),
    "dpso_bound_fallbacks": (_I32, [_P]),
    "dpso_band_runs": (_I32, [_P]),
    "dpso_bound_pairs": (_I32, [_P, _P]),
    "dpso_band_line": (_I32, [_P]),
    "dpso_band_rows": (_I32, [_P]),
    "dpso_step_timed": (_I32, [_P, _I32, _P, _P]),
    "dpso_ctl": (_I32, [_P, _P, _P]),
    "dpso_result": (_I32, [_P, _P, _P, _P, ctypes.POINTER(_I32)]),
    "dpso_get_state": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "dpso_set_state": (_I32, [_P, _P, _P, _P, _P, _P, _P, ctypes.c_double]),
    "dpso_offer_gbest": (_I32, [_P, _P, ctypes.c_double]),
    "dpso_mutate_step": (_I32, [_P]),
    "dpso_scan_chunks": (_I32, [_I32, _I32]),
    "dpso_island_record_bytes": (_I64, [_I32]),
    "dpso_island_pack": (_I32, [_P, _P, _I32]),
    "dpso_island_adopt": (_I32, [_P, _P, _I32, _I32]),
    "dpso_destroy": (None, [_P]),
    "dpso_last_error": (ctypes.c_char_p, []),
    "dpso_tour_cost_batch": (_I32, [_P, _I64, _I32, _P, _I32, _P, _P]),
    "dpso_best_exchange_batch": (_I32, [_P, _I64, _I32, _P, _I32, _P, _P]),
    "dpso_nn_tour": (_I32, [_P, _I64, _I32, _I32, _P, _P]),
    "dpso_nn_two_opt": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "dpso_build_cost": (_I32, [_P, _I32, _I32, _I32, _P, _P, _I32, _P, _I64,
                                _P, _P, _P]),
    "dpso_build_cost_rows": (_I32, [_P, _I32, _I32, _I32, _P, _P, _I32, _I32,
                                     _I32, _P, _P]),
    "dpso_build_cost_assemble": (_I32, [_P, _I32, _P, _I64, _P, _P, _P]),
    "dpso_philox4x32_10": (_I32, [_P, ctypes.c_uint64, _P]),
    "dpso_upload_matrix": (_I32, [_P, _I64, _I32, _I32, _P, _I64, _P]),
    "dpso_write_matrix_text": (_I32, [ctypes.c_char_p, _P, _I64, _I32]),
    "dpso_read_matrix_text": (_I32, [ctypes.c_char_p, _P, _I64, _I32,
                                     ctypes.POINTER(_I32)]),
    "dpso_py_repr": (_I32, [ctypes.c_double, ctypes.c_char_p, _I32]),
    "dpso_spawn_pcg64_states": (_I32, [_P, _I32, _I64, _P]),
    "dpso_voxel_paths": (_I32, [_P, _I32, _I32, _I32, _P, _I32, _P, _I32,
                                _P, _I64, _P, _P]),
    "dpso_version": (ctypes.c_char_p, []),
}
EXPORTED = tuple(_SIG)

_lock = threading.Lock()
_lib = None


class DpsoError(RuntimeError):
    pass


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library (no CUDA calls are made by loading)."""
    global _lib
    with _lock:
        if _lib is not None and path == LIB_PATH:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: the CUDA extension is not built "
                "(run `python -m paper_1706_04399_b200.build`); there is no "
                "CPU fallback")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIG.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path == LIB_PATH:
            _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == DPSO_OK:
        return
    msg = (load().dpso_last_error() or b"").decode()
    if rc == DPSO_EINVAL:
        raise ValueError(msg)
    raise DpsoError(msg)
