"""Plain-text cost-matrix I/O (graph.py:123-143) in native host code: the
writer's bytes equal the reference's (restated in oracle/graph_oracle.py),
the reader returns the same values and raises the same errors.  Host-only
entry points of libdpso.so: no GPU needed."""
import ctypes
import struct

import numpy as np
import pytest

from oracle import graph_oracle as G


@pytest.fixture(scope="module")
def pkg():
    from paper_1706_04399_b200.build import build
    build()
    import paper_1706_04399_b200 as pkg
    return pkg


def py_repr_native(lib, x):
    buf = ctypes.create_string_buffer(64)
    assert lib.dpso_py_repr(x, buf, 64) == 0
    return buf.value.decode()


def interesting_doubles(rng, k):
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 0.1, 0.2, 0.3, 1e16, 1e15, 9.999e15,
            1e-4, 1e-5, 0.0001, 0.00011, 123456789012345678.0, 1e22, 1e-300,
            5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
            float("inf"), float("-inf"), float("nan"), 2.0 ** 53,
            2.0 ** 53 + 2, 1 / 3, 2 / 3, 100.0, 1234.5, 44.0, 1e6, 1e7,
            816000.0, 3.14159e-7]
    vals += list(rng.random(k) * 10.0)
    vals += list(np.floor(rng.random(k) * 2000.0))
    vals += list(np.exp(rng.uniform(-700, 700, k)))
    bits = rng.integers(0, 2 ** 63, k, dtype=np.int64)
    vals += [struct.unpack("<d", struct.pack("<q", int(b)))[0] for b in bits]
    return vals


def test_py_repr_matches_python(pkg):
    from paper_1706_04399_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(5)
    for x in interesting_doubles(rng, 3000):
        assert py_repr_native(lib, x) == repr(float(x)), x


def test_save_is_byte_identical(pkg, tmp_path):
    rng = np.random.default_rng(7)
    for n in (0, 1, 2, 15, 57):
        cost = rng.random((n, n)) * 10.0 ** float(rng.integers(-6, 9))
        if n > 3:
            cost[0, 1] = 1e6
            cost[1, 0] = float("inf")
            cost[2, 2] = -0.0
        a, b = tmp_path / f"ours{n}.txt", tmp_path / f"ref{n}.txt"
        pkg.save_cost_matrix(a, cost)
        G.save_cost_matrix(b, cost)
        assert a.read_bytes() == b.read_bytes(), n


def test_load_matches_reference(pkg, tmp_path):
    rng = np.random.default_rng(9)
    cost = np.floor(rng.random((40, 40)) * 100) + rng.random((40, 40))
    p = tmp_path / "m.txt"
    G.save_cost_matrix(p, cost)
    got = pkg.load_cost_matrix(p)
    ref = G.load_cost_matrix(p)
    assert got.dtype == np.float64 and got.shape == (40, 40)
    assert np.array_equal(got.view(np.int64), ref.view(np.int64))
    # free-form whitespace, signs, underscores, inf/nan, exponents
    p.write_text("  3\n\t1_000 +2.5 -0.0\n1E3 .5 5. \f\v inf -Infinity nan\n")
    got, ref = pkg.load_cost_matrix(p), G.load_cost_matrix(p)
    assert np.array_equal(np.nan_to_num(got), np.nan_to_num(ref))
    assert np.isnan(got[2, 2]) and np.signbit(got[0, 2])


@pytest.mark.parametrize("text", [
    "", "   \n", "x\n", "2\n1 2 3\n", "2\n1 2 3 4 5\n", "2\n1 2 z 4\n",
    "2\n1 2 3 1__0\n", "1.0\n1\n", "2\n1 2 3 _4\n",
])
def test_load_errors_match_reference(pkg, tmp_path, text):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(ValueError) as ref:
        G.load_cost_matrix(p)
    with pytest.raises(ValueError) as ours:
        pkg.load_cost_matrix(p)
    assert str(ours.value) == str(ref.value)


def test_missing_file(pkg, tmp_path):
    with pytest.raises(FileNotFoundError):
        pkg.load_cost_matrix(tmp_path / "nope.txt")
