"""The numpy-RNG restatement (oracle/np_random.py) equals the installed numpy
bit for bit, for every draw the reference makes (solver.py:180-250)."""
import numpy as np
import pytest

from oracle.np_random import PCG64Stream


@pytest.mark.parametrize("seed", range(12))
def test_draw_sequences_match_numpy(seed):
    ss = np.random.SeedSequence(seed).spawn(2)
    g = np.random.Generator(np.random.PCG64(ss[0]))
    s = PCG64Stream.from_generator(g)
    rs = np.random.RandomState(seed)
    for _ in range(40):
        op = rs.randint(5)
        n = int(rs.choice([2, 3, 4, 5, 7, 16, 100, 1000, 1001, 9999, 10000,
                           10001, 20000, 70000]))
        if op == 0:
            assert list(g.random(2)) == list(s.random2())
        elif op == 1:
            m = min(n, 2000)
            assert [int(v) for v in g.permutation(m)] == s.permutation(m)
        elif op == 2:
            sz = int(rs.randint(1, min(n, 600) + 1))
            assert ([int(v) for v in g.choice(n, size=sz, replace=False)]
                    == s.choice_noreplace(n, sz))
        elif op == 3:
            hi = max(2, n // 4)
            assert int(g.integers(1, hi + 1)) == s.integers(1, hi + 1)
        else:
            assert ([int(v) for v in g.choice(n, size=2, replace=False)]
                    == s.choice_noreplace(n, 2))
    st = g.bit_generator.state
    assert st["state"]["state"] == s.state
    assert st["has_uint32"] == s.has_uint32


def test_lemire_rejection_path():
    # ranges close to 2**32 make rejection likely; exercise the retry loop
    g = np.random.Generator(np.random.PCG64(7))
    s = PCG64Stream.from_generator(g)
    for hi in (2**32 - 7, 3 * 2**30 + 1, 2**31 + 5):
        for _ in range(200):
            assert int(g.integers(0, hi)) == s.integers(0, hi)
