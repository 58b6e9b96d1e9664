"""The C-ABI library builds for sm_100a, loads on a CPU host, and exports
every symbol include/dpso.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1706_04399_b200 import _lib
from paper_1706_04399_b200.build import build


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dpso.h")).read()
    return sorted(set(re.findall(r"\b(dpso_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_lib.EXPORTED)


def test_version_and_param_validation(lib):
    assert b"sm_100a" in lib.dpso_version()
    p = _lib.DpsoParams(n_particles=2, inertia=1.0, cognitive=0.4,
                        social=0.4, max_generations=10, stall_generations=5,
                        mutation_period=3, seed_fraction=0.1, use_mutation=1,
                        use_edge_exchange=1, parallel=0, rng_mode=0)
    nb = ctypes.c_size_t(0)
    rc = lib.dpso_workspace_size(ctypes.byref(p), 10, ctypes.byref(nb))
    assert rc == _lib.DPSO_EINVAL
    assert b"n_particles must be >= 3" in lib.dpso_last_error()
    with pytest.raises(ValueError, match="n_particles"):
        _lib.check(rc)
    p.n_particles = 32
    p.inertia = 1.5
    rc = lib.dpso_workspace_size(ctypes.byref(p), 10, ctypes.byref(nb))
    assert rc == _lib.DPSO_EINVAL and b"inertia" in lib.dpso_last_error()
    p.inertia = 1.0
    assert lib.dpso_workspace_size(ctypes.byref(p), 1000,
                                   ctypes.byref(nb)) == 0
    assert nb.value > 32 * 1000 * 2 * 3


def test_sass_is_sm100a():
    so = os.path.join(ROOT, "paper_1706_04399_b200", "libdpso.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out


def test_estimator_api_cpu():
    # construction / get_params / validation never touch the device
    from paper_1706_04399_b200 import DiscreteSwarmSolver
    s = DiscreteSwarmSolver(n_particles=10, random_state=5)
    params = s.get_params()
    assert params["n_particles"] == 10
    assert DiscreteSwarmSolver(**params).get_params() == params
    s.set_params(social=0.3)
    assert s.social == 0.3
    import numpy as np
    with pytest.raises(ValueError):
        DiscreteSwarmSolver().fit(np.zeros((3, 2)))
    with pytest.raises(ValueError):
        DiscreteSwarmSolver(n_particles=2).fit(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        DiscreteSwarmSolver(mutation_period=0).fit(np.zeros((3, 3)))
    r = DiscreteSwarmSolver(random_state=0).fit(np.zeros((1, 1)))
    assert r.best_tour_ == (0, 0) and r.n_generations_ == 1


def test_philox_known_answers(lib):
    # Random123 kat_vectors for philox4x32_10
    import numpy as np
    kats = [
        ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
        ((0xffffffff,) * 4, (0xffffffff, 0xffffffff),
         (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
        ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344),
         (0xa4093822, 0x299f31d0),
         (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
    ]
    for ctr, key, want in kats:
        c = np.array(ctr, dtype=np.uint32)
        out = np.zeros(4, dtype=np.uint32)
        rc = lib.dpso_philox4x32_10(c.ctypes.data_as(ctypes.c_void_p),
                                    key[0] | (key[1] << 32),
                                    out.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        assert tuple(int(v) for v in out) == want


def test_stream_states_match_numpy_seedsequence():
    """The vectorised SeedSequence.spawn -> PCG64 restatement used to seed
    the device streams equals numpy's own, for one- and multi-word seeds."""
    import numpy as np
    from paper_1706_04399_b200.solver import _spawned_pcg64_states
    m = (1 << 64) - 1
    for seed in (0, 1, 7, 2923, 2**32 - 1, 2**32, 2**32 + 5, 2**70 + 3):
        for count in (1, 5, 130):
            want = np.empty((count, 6), dtype=np.uint64)
            for i, s in enumerate(np.random.SeedSequence(seed).spawn(count)):
                st = np.random.PCG64(s).state
                a, b = st["state"]["state"], st["state"]["inc"]
                want[i] = (a >> 64, a & m, b >> 64, b & m, st["has_uint32"],
                           st["uinteger"])
            got = _spawned_pcg64_states(seed, count)
            assert np.array_equal(got, want), (seed, count)


def test_native_stream_states_match_numpy():
    """dpso_spawn_pcg64_states (host code, threaded) equals numpy's
    SeedSequence.spawn -> PCG64, including counts that cross its thread
    chunks and multi-word seeds."""
    import numpy as np
    from paper_1706_04399_b200.solver import (_spawned_pcg64_states,
                                              numpy_stream_states)
    m = (1 << 64) - 1
    for seed in (0, 7, 2923, 2**32 + 5, 2**70 + 3, 2**128 + 11):
        for count in (1, 130):
            want = np.empty((count, 6), dtype=np.uint64)
            for i, s in enumerate(np.random.SeedSequence(seed).spawn(count)):
                st = np.random.PCG64(s).state
                a, b = st["state"]["state"], st["state"]["inc"]
                want[i] = (a >> 64, a & m, b >> 64, b & m, st["has_uint32"],
                           st["uinteger"])
            assert np.array_equal(numpy_stream_states(seed, count), want)
    big = numpy_stream_states(1000, 20000)  # several threads
    assert np.array_equal(big, _spawned_pcg64_states(1000, 20000))
