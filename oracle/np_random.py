"""Restatement of the numpy random primitives the reference solver draws from.

TEST INFRASTRUCTURE ONLY — this module is the checker, never the product.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg may import it.

The reference (``/root/reference/pkg/src/inspectour/solver.py:278-282``) seeds
``np.random.SeedSequence(random_state).spawn(P + 2)`` and wraps every child in
``np.random.Generator(np.random.PCG64(...))``.  The draws it consumes are:

* ``Generator.random(2)``           (solver.py:191)   -> ``next_double`` x2
* ``Generator.choice(n, 2, replace=False)`` (solver.py:180) -> Floyd + shuffle
* ``Generator.permutation(n)``      (solver.py:183)   -> masked-interval shuffle
* ``Generator.integers(1, k_hi+1)`` (solver.py:246)   -> Lemire bounded uint32
* ``Generator.choice(n, 2k, replace=False)`` (solver.py:250)

Third-party dependency: numpy (installed here: 2.3.5; the reference pins only
``numpy>=1.24``, ``pyproject.toml:10-14``).  The algorithms restated below are
numpy's published ones: PCG64 = PCG XSL-RR 128/64 (``numpy/random/src/pcg64``),
``random_bounded_uint64`` / ``buffered_bounded_lemire_uint32`` /
``random_interval`` (``numpy/random/src/distributions/distributions.c``),
Floyd's sampler and ``_shuffle_int`` / ``_shuffle_raw``
(``numpy/random/_generator.pyx``).  Bit-equality with the installed numpy is
pinned by ``tests/test_oracle_rng.py`` over many seeds and sizes; the CUDA
device implementation (``paper_1706_04399_b200/csrc/pcg64.cuh``) restates the
same algorithms and is pinned against this module and against numpy.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


class PCG64Stream:
    """numpy ``PCG64`` bit generator state + the ``Generator`` draws we need."""

    def __init__(self, state: int, inc: int, has_uint32: int = 0,
                 uinteger: int = 0):
        self.state = state & MASK128
        self.inc = inc & MASK128
        self.has_uint32 = has_uint32
        self.uinteger = uinteger
        self.n64 = 0  # 64-bit outputs consumed (for cursor bookkeeping)

    @classmethod
    def from_seed_sequence(cls, seq) -> "PCG64Stream":
        st = np.random.PCG64(seq).state
        return cls(st["state"]["state"], st["state"]["inc"],
                   st["has_uint32"], st["uinteger"])

    @classmethod
    def from_generator(cls, gen: np.random.Generator) -> "PCG64Stream":
        st = gen.bit_generator.state
        return cls(st["state"]["state"], st["state"]["inc"],
                   st["has_uint32"], st["uinteger"])

    # -- raw outputs ---------------------------------------------------------
    def next64(self) -> int:
        self.state = (self.state * PCG_MULT + self.inc) & MASK128
        s = self.state
        x = ((s >> 64) ^ s) & MASK64
        rot = s >> 122
        self.n64 += 1
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next32(self) -> int:
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        v = self.next64()
        self.has_uint32 = 1
        self.uinteger = v >> 32
        return v & 0xFFFFFFFF

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    # -- bounded integers ----------------------------------------------------
    def lemire32(self, rng: int) -> int:
        """``buffered_bounded_lemire_uint32``: uniform in [0, rng]."""
        rng_excl = rng + 1
        m = self.next32() * rng_excl
        leftover = m & 0xFFFFFFFF
        if leftover < rng_excl:
            threshold = (0xFFFFFFFF - rng) % rng_excl
            while leftover < threshold:
                m = self.next32() * rng_excl
                leftover = m & 0xFFFFFFFF
        return m >> 32

    def bounded(self, rng: int) -> int:
        """``random_bounded_uint64(state, 0, rng, 0, use_masked=False)``."""
        if rng == 0:
            return 0
        if rng <= 0xFFFFFFFF:
            if rng == 0xFFFFFFFF:
                return self.next32()
            return self.lemire32(rng)
        raise NotImplementedError("64-bit ranges never occur for N < 2**32")

    def interval(self, mx: int) -> int:
        """``random_interval``: masked rejection, uniform in [0, mx]."""
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= 0xFFFFFFFF:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    # -- Generator methods ---------------------------------------------------
    def random2(self) -> tuple[float, float]:
        return self.next_double(), self.next_double()

    def integers(self, low: int, high: int) -> int:
        """``Generator.integers(low, high)`` scalar int64, endpoint=False."""
        return low + self.bounded(high - 1 - low)

    def permutation(self, n: int) -> list[int]:
        arr = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            arr[i], arr[j] = arr[j], arr[i]
        return arr

    def choice_noreplace(self, n: int, size: int) -> list[int]:
        """``Generator.choice(n, size, replace=False)`` (shuffle=True)."""
        if size > n:
            raise ValueError("size > n")
        cutoff = 50
        if n > 10000 and size > n // cutoff:
            # tail shuffle: _shuffle_int(n, max(n - size, 1), arange(n))
            idx = list(range(n))
            for i in range(n - 1, max(n - size, 1) - 1, -1):
                j = self.bounded(i)
                idx[i], idx[j] = idx[j], idx[i]
            return idx[n - size:]
        # Floyd's algorithm, then _shuffle_int(size, 1, idx)
        out = [0] * size
        seen = set()
        for t, j in enumerate(range(n - size, n)):
            val = self.bounded(j)
            if val in seen:
                val = j
            seen.add(val)
            out[t] = val
        for i in range(size - 1, 0, -1):
            j = self.bounded(i)
            out[i], out[j] = out[j], out[i]
        return out
