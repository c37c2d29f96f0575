"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's static-noise draw.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg may import this module, and only as the checker.  The product path draws
noise on the device (``csrc/noise.cu``) and never calls into ``oracle/``.

What it restates
----------------
``ctqw.noise.init_process`` (``pkg/src/ctqw/noise.py:128-159``) draws, per
realization ``r``,

    rng = np.random.default_rng((master_seed, r))        # ensemble.py:680-682
    values = rng.choice(levels, size=n_links + n_sites)   # noise.py:150-154

The arithmetic lives in NumPy (third-party, not vendored under
/root/reference; this container has numpy 2.3.5, the reference pins only
``numpy>=1.24`` in ``pkg/pyproject.toml:11``).  Its published algorithm is:

* ``SeedSequence`` entropy mixing with a 4-word pool
  (numpy/random/bit_generator.pyx: ``mix_entropy``, ``generate_state``);
* ``PCG64`` = 128-bit LCG, XSL-RR 64-bit output, seeded from
  ``generate_state(4, uint64)`` (numpy/random/src/pcg64/pcg64.{h,c});
* ``Generator.choice(a, size)`` with ``replace=True, p=None`` =
  ``integers(0, len(a), size, dtype=int64)`` -> ``random_bounded_uint64_fill``
  -> 32-bit Lemire rejection on ``next_uint32`` (numpy/random/src/
  distributions/distributions.c: ``buffered_bounded_lemire_uint32``), which
  for PCG64 hands out the low half of each 64-bit output first, then the high
  half cached in the bit generator.  The cache persists across calls; for the
  static draw (one call on a fresh generator) ``bounded_indices`` below
  models it locally.

Pinned by ``tests/test_oracle_golden.py`` against draws produced by the
reference's own ``init_process`` (fixtures in ``tests/golden/``).
"""

from __future__ import annotations

import numpy as np

MASK32 = 0xFFFFFFFF
MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1

INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
XSHIFT = 16
POOL_SIZE = 4

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _uint32_words(value: int) -> list[int]:
    """Little-endian 32-bit words of a non-negative int (0 -> [0])."""
    if value < 0:
        raise ValueError("seed words must be non-negative")
    if value == 0:
        return [0]
    words = []
    while value:
        words.append(value & MASK32)
        value >>= 32
    return words


def seed_pool(entropy) -> list[int]:
    """SeedSequence(entropy).pool for a tuple of non-negative ints."""
    words = [w for v in entropy for w in _uint32_words(int(v))]
    hash_const = INIT_A

    def hashmix(value: int) -> int:
        nonlocal hash_const
        value = (value ^ hash_const) & MASK32
        hash_const = (hash_const * MULT_A) & MASK32
        value = (value * hash_const) & MASK32
        return value ^ (value >> XSHIFT)

    def mix(x: int, y: int) -> int:
        out = (MIX_MULT_L * x - MIX_MULT_R * y) & MASK32
        return out ^ (out >> XSHIFT)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(POOL_SIZE)]
    for src in range(POOL_SIZE):
        for dst in range(POOL_SIZE):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(POOL_SIZE, len(words)):
        for dst in range(POOL_SIZE):
            pool[dst] = mix(pool[dst], hashmix(words[src]))
    return pool


def generate_state_u64(pool: list[int], n_words: int = 4) -> list[int]:
    """SeedSequence.generate_state(n_words, np.uint64)."""
    hash_const = INIT_B
    out32 = []
    for i in range(2 * n_words):
        value = pool[i % len(pool)]
        value = (value ^ hash_const) & MASK32
        hash_const = (hash_const * MULT_B) & MASK32
        value = (value * hash_const) & MASK32
        value ^= value >> XSHIFT
        out32.append(value)
    return [out32[2 * k] | (out32[2 * k + 1] << 32) for k in range(n_words)]


class Pcg64:
    """PCG64 (XSL-RR 128/64) seeded the way ``np.random.PCG64(SeedSequence)`` is."""

    def __init__(self, entropy):
        s = generate_state_u64(seed_pool(entropy), 4)
        initstate = (s[0] << 64) | s[1]
        initseq = (s[2] << 64) | s[3]
        self.inc = ((initseq << 1) | 1) & MASK128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & MASK128
        self._step()

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & MASK128

    def next64(self) -> int:
        self._step()
        rot = self.state >> 122
        x = ((self.state >> 64) ^ self.state) & MASK64
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64


def bounded_indices(gen: Pcg64, n_levels: int, count: int) -> list[int]:
    """``Generator.integers(0, n_levels, count)`` via buffered 32-bit Lemire."""
    rng = n_levels - 1
    if rng == 0:
        return [0] * count
    excl = rng + 1
    buf = 0
    have = 0
    out = []

    def next32():
        nonlocal buf, have
        if have == 0:
            buf = gen.next64()
            have = 1
            return buf & MASK32
        have = 0
        return (buf >> 32) & MASK32

    for _ in range(count):
        m = next32() * excl
        leftover = m & MASK32
        if leftover < excl:
            threshold = (MASK32 - rng) % excl
            while leftover < threshold:
                m = next32() * excl
                leftover = m & MASK32
        out.append(m >> 32)
    return out


def draw_static_noise(master_seed: int, realization: int, levels, total: int) -> np.ndarray:
    """One realization's ``values`` array of ``init_process`` (noise.py:150-154)."""
    levels = np.asarray(levels, dtype=np.float64)
    idx = bounded_indices(Pcg64((master_seed, realization)), len(levels), total)
    return levels[np.asarray(idx, dtype=np.int64)] if total else np.empty(0)


def draw_static_noise_stack(master_seed: int, r0: int, count: int, levels, total: int) -> np.ndarray:
    """``(count, total)`` stack for realizations ``r0 .. r0+count-1``."""
    out = np.empty((count, total), dtype=np.float64)
    for i in range(count):
        out[i] = draw_static_noise(master_seed, r0 + i, levels, total)
    return out


class TelegraphOracle:
    """Dynamic telegraph noise of a batch of realizations (TEST ONLY).

    Restates ``init_process`` / ``advance`` (``pkg/src/ctqw/noise.py:128-206``)
    for ``rate > 0``.  The arithmetic of those functions is NumPy's
    ``Generator`` (``choice`` and ``exponential``, the ziggurat sampler of
    numpy/random/src/distributions/distributions.c); it is called here as
    the reference calls it, with one ``default_rng((master_seed, r))`` per
    realization (``ensemble.py:680-682``), so this is the reference algorithm
    on the same streams.  ``values``/``next_switch`` are laid out
    ``[links | sites]`` per realization.
    """

    def __init__(self, master_seed, r0, count, levels, n_links, n_sites, rate):
        self.levels = np.asarray(levels, dtype=np.float64)
        self.n_links, self.n_sites = int(n_links), int(n_sites)
        total = self.n_links + self.n_sites
        self.mean_wait = 1.0 / float(rate)
        self.rngs = [np.random.default_rng((int(master_seed), int(r))) for r in range(r0, r0 + count)]
        self.values = np.empty((count, total))
        self.next_switch = np.empty((count, total))
        for i, g in enumerate(self.rngs):          # noise.py:152-157
            self.values[i] = g.choice(self.levels, size=total)
            self.next_switch[i] = g.exponential(1.0 / float(rate), size=total)
        self.time = np.zeros(count)
        self.switches = np.zeros(count, dtype=np.int64)

    def advance(self, dt):
        """``advance(process, dt)`` for every realization (noise.py:175-206)."""
        for i, g in enumerate(self.rngs):
            t_end = self.time[i] + dt
            due = self.next_switch[i] <= t_end
            if self.values.shape[1] and due.any():
                idx = np.nonzero(due)[0]
                while idx.size:
                    self.switches[i] += idx.size
                    self.values[i, idx] = g.choice(self.levels, size=idx.size)
                    self.next_switch[i, idx] += g.exponential(self.mean_wait, size=idx.size)
                    idx = idx[self.next_switch[i, idx] <= t_end]
            self.time[i] = t_end

    def link_values(self):
        return self.values[:, : self.n_links]

    def site_values(self):
        return self.values[:, self.n_links:]
