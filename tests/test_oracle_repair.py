"""The data-parallel prefix-repair formulation used by the CUDA update kernel
(oracle.dpso_oracle.sigma_prefix) equals the reference's sequential
left-to-right repair + prefix truncation (solver.py:57-69, 82-85)."""
import itertools
import random

from oracle.dpso_oracle import apply_open, prefix_len, sigma_prefix, \
    subtract_open


def expected_sigma(x, T, c):
    t = subtract_open(T, x)
    k = prefix_len(c, len(t))
    cur = apply_open(x, t[:k])
    sig = list(range(len(x)))
    for q, v in enumerate(x):
        sig[v] = cur[q]
    return sig, k, len(t)


def test_exhaustive_small():
    for n in range(1, 6):
        perms = list(itertools.permutations(range(n)))
        for x in perms:
            for T in perms:
                L = len(subtract_open(list(T), list(x)))
                for k in range(L + 1):
                    c = k / L if L else 0.5
                    assert sigma_prefix(list(x), list(T), c) == \
                        expected_sigma(list(x), list(T), c)


def test_random_large():
    rng = random.Random(5)
    for _ in range(400):
        n = rng.randint(2, 400)
        x = list(range(n))
        T = list(range(n))
        rng.shuffle(x)
        rng.shuffle(T)
        c = rng.random()
        assert sigma_prefix(x, T, c) == expected_sigma(x, T, c)
