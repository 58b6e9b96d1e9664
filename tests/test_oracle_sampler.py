"""The data-parallel formulation of numpy's choice(n, 2k, replace=False)
(Floyd's sampler, then _shuffle_int) used by k_mut_sample
(k_mutate.cu: floyd_shuffle_warp) equals the sequential algorithm the
reference's _mutate consumes (solver.py:236-238, numpy
_generator.pyx choice / _shuffle_int), for every draw sequence - checked
here on CPU over random draws, including n == 2k (the j == 0 step takes
no draw)."""
import random


def sequential(vals, n, size):
    chosen, out, d = set(), [], 0
    for t in range(size):
        j = n - size + t
        if j == 0:
            val = 0
        else:
            val = vals[d]
            d += 1
        if val in chosen:
            val = j
        chosen.add(val)
        out.append(val)
    for i in range(size - 1, 0, -1):
        j = vals[d]
        d += 1
        out[i], out[j] = out[j], out[i]
    return out


def parallel(vals, n, size):
    """floyd_shuffle_warp, lane loops written as plain loops."""
    nmz = n - size
    zero = 1 if nmz == 0 else 0
    F = size - zero

    def vt(t):
        return 0 if (zero and t == 0) else vals[t - zero]

    first = {}
    for t in range(size):  # atomicMin: the first step to draw each value
        first[vt(t)] = min(first.get(vt(t), size), t)
    col = [first[vt(t)] < t for t in range(size)]
    while True:  # col(t) |= col(v_t - nmz) for an earlier collided step
        changed = False
        for t in range(size):
            v = vt(t)
            if not col[t] and v >= nmz and v - nmz < t and col[v - nmz]:
                col[t] = changed = True
        if not changed:
            break
    sidx = [nmz + t if col[t] else vt(t) for t in range(size)]
    writers = {}
    for i in range(1, size):  # step i writes position w_i
        writers.setdefault(vals[F + size - 1 - i], []).append(i)

    def above(x, y):
        c = [w for w in writers.get(x, []) if w > y]
        return min(c) if c else None

    out = []
    for i in range(size):
        x = 0 if i == 0 else vals[F + size - 1 - i]
        w = above(x, i)
        while w is not None:
            x = w
            w = above(x, x)
        out.append(sidx[x])
    return out


def draws(rng, n, size):
    vals = [rng.randint(0, n - size + t) for t in range(size)
            if n - size + t != 0]
    vals += [rng.randint(0, i) for i in range(size - 1, 0, -1)]
    return vals


def test_parallel_sampler_equals_sequential():
    rng = random.Random(7)
    for _ in range(20000):
        n = rng.randint(2, 80)
        kmax = min(max(2, n // 4), n // 2)
        size = 2 * rng.randint(1, kmax)
        vals = draws(rng, n, size)
        assert parallel(vals, n, size) == sequential(vals, n, size)


def test_full_size_events():
    # n == 2k: Floyd's first step is j = 0 (no draw)
    rng = random.Random(8)
    for n in (2, 4, 6, 8):
        for _ in range(2000):
            vals = draws(rng, n, n)
            assert parallel(vals, n, n) == sequential(vals, n, n)


def test_large_events():
    rng = random.Random(9)
    for n in (1000, 2000):
        for _ in range(20):
            size = 2 * rng.randint(1, n // 4)
            vals = draws(rng, n, size)
            assert parallel(vals, n, size) == sequential(vals, n, size)
