import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1706_04399_b200 import DiscreteSwarmSolver, _lib
from paper_1706_04399_b200.solver import device_cost, SwarmContext, numpy_stream_states
n, P = 1000, 1024
rng = np.random.default_rng(1000)
pts = rng.random((n, 2)) * 10.0
cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1)); np.fill_diagonal(cost, 0.0)
s = DiscreteSwarmSolver(n_particles=P, max_generations=20, stall_generations=20, random_state=7)
s.fit(cost)
for rep in range(3):
    T = {}
    def tick(k, t0):
        torch.cuda.synchronize(); T[k] = round((time.perf_counter() - t0) * 1e3, 2); return time.perf_counter()
    t = time.perf_counter()
    c = s._check_cost(cost); t = tick('check', t)
    ct, ld = device_cost(c); t = tick('device_cost', t)
    params = s._params()
    lib = _lib.load()
    nb = ctypes.c_size_t(0); lib.dpso_workspace_size(ctypes.byref(params), n, ctypes.byref(nb)); t = tick('ws_size', t)
    ws = torch.empty(int(nb.value), dtype=torch.uint8, device='cuda'); t = tick('ws_alloc', t)
    h = ctypes.c_void_p()
    _lib.check(lib.dpso_create(ctypes.byref(params), n, ws.data_ptr(), int(nb.value), torch.cuda.current_stream().cuda_stream, ctypes.byref(h))); t = tick('create', t)
    _lib.check(lib.dpso_set_cost(h, ct.data_ptr(), ld)); t = tick('set_cost', t)
    st = numpy_stream_states(7, P + 2); t = tick('seedseq', t)
    _lib.check(lib.dpso_set_streams(h, np.ascontiguousarray(st, dtype=np.uint64).ctypes.data_as(ctypes.c_void_p))); t = tick('set_streams', t)
    _lib.check(lib.dpso_init(h, None, 0)); t = tick('init', t)
    g = ctypes.c_int32(0); _lib.check(lib.dpso_run(h, ctypes.byref(g))); t = tick('run20', t)
    lib.dpso_destroy(h); t = tick('destroy', t)
    del ws; t = tick('free', t)
    print(T)
