"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the seeded random
budget fill ``np.random.default_rng(rng_seed).choice(pool, fill_n,
replace=False)`` (reference pkg/src/flashfps/fps_prune.py:101-103).

The arithmetic lives in NumPy (third-party, not vendored in the reference;
pinned by the reference only as ``numpy>=1.24``, pkg/pyproject.toml:10; this
image carries NumPy 2.3.5).  Restated from NumPy's published algorithm:

* ``PCG64`` (PCG XSL-RR 128/64): state <- state * M + inc, then output
  rotr64(hi ^ lo, hi >> 58); 32-bit draws take the low half of one output and
  buffer the high half for the next draw (``pcg64_next32``).
* ``random_bounded_uint64(0, rng)`` for rng < 2^32 - 1: Lemire's multiply-
  shift on one 32-bit draw with rejection below (2^32 - 1 - rng) % (rng + 1).
* ``Generator.choice(a, size, replace=False)`` without p: when
  pop > 10000 and size > pop // 50, a partial Fisher-Yates of arange(pop) from
  the tail (``_shuffle_int(pop, max(pop - size, 1))``) keeping the last `size`
  entries; otherwise Floyd's algorithm over a linear-probing hash set of
  (1 + mask) slots, mask = the smallest 2^k - 1 >= uint64(1.2 * size), followed
  by ``_shuffle_int(size, 1)`` of the picks.  The result is ``a[idx]``.

The initial PCG64 state comes from ``np.random.PCG64(seed).state`` (the
SeedSequence hashing is set-up, not sampling).  tests/test_npchoice.py pins
this restatement against NumPy's own output; the CUDA fill (csrc/fill.cu)
follows it step by step and is checked against both.
"""

from __future__ import annotations

M128 = (2549297995355413924 << 64) | 4865540595714422341
MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1


def pcg64_seed_state(seed: int) -> tuple[int, int]:
    """(state, inc) of np.random.PCG64(seed) — the one NumPy call used."""
    import numpy as np
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


class PCG64:
    def __init__(self, state: int, inc: int):
        self.s, self.inc = state, inc
        self.has32, self.buf32 = False, 0
        self.rejections = 0  # Lemire redraws (tests check the path is exercised)

    def next64(self) -> int:
        self.s = (self.s * M128 + self.inc) & MASK128
        hi, lo = self.s >> 64, self.s & MASK64
        x, r = hi ^ lo, hi >> 58
        return ((x >> r) | (x << (64 - r))) & MASK64 if r else x

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.buf32
        v = self.next64()
        self.has32, self.buf32 = True, v >> 32
        return v & 0xFFFFFFFF

    def bounded(self, rng: int) -> int:
        """random_bounded_uint64(off=0, rng, mask=0, use_masked=False), rng < 2^32."""
        if rng == 0:
            return 0
        if rng == 0xFFFFFFFF:
            return self.next32()
        assert rng < 0xFFFFFFFF
        excl = rng + 1
        m = self.next32() * excl
        left = m & 0xFFFFFFFF
        if left < excl:
            thr = (0xFFFFFFFF - rng) % excl
            while left < thr:
                self.rejections += 1
                m = self.next32() * excl
                left = m & 0xFFFFFFFF
        return m >> 32


def _shuffle_int(g: PCG64, n: int, first: int, data: list) -> None:
    for i in range(n - 1, first - 1, -1):
        j = g.bounded(i)
        data[i], data[j] = data[j], data[i]


def choice_idx(pop: int, size: int, state: int, inc: int, gen: PCG64 | None = None) -> list:
    """Positions (into the pool) Generator.choice(pool, size, replace=False)
    returns, for a generator in PCG64 state (state, inc)."""
    g = gen if gen is not None else PCG64(state, inc)
    if size == 0:
        return []
    if pop > 10000 and size > pop // 50:
        data = list(range(pop))
        _shuffle_int(g, pop, max(pop - size, 1), data)
        return data[pop - size:]
    set_size = int(1.2 * size)
    mask = set_size
    for sh in (1, 2, 4, 8, 16, 32):
        mask |= mask >> sh
    empty = MASK64
    hs = [empty] * (mask + 1)
    out = []
    for j in range(pop - size, pop):
        val = g.bounded(j)
        loc = val & mask
        while hs[loc] != empty and hs[loc] != val:
            loc = (loc + 1) & mask
        if hs[loc] == empty:
            hs[loc] = val
            out.append(val)
        else:
            loc = j & mask
            while hs[loc] != empty:
                loc = (loc + 1) & mask
            hs[loc] = j
            out.append(j)
    _shuffle_int(g, size, 1, out)
    return out


def seeded_fill(order_k, n: int, fill_n: int, rng_seed: int) -> list:
    """fps_prune.py:96-103 with FillMode.SEEDED_RANDOM: the pool is the
    ascending complement of the kernel's picks in [0, n)."""
    picked = set(int(v) for v in order_k)
    pool = [i for i in range(n) if i not in picked]
    st, inc = pcg64_seed_state(rng_seed)
    return [pool[i] for i in choice_idx(len(pool), fill_n, st, inc)]
