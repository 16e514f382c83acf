"""Oracle: the NumPy PCG64 / Generator recipes the device RNG must replay.

NumPy PCG64 (numpy/random/src/pcg64): 128-bit LCG state, advance-then-output
XSL-RR.  Generator.uniform = (raw >> 11) * 2**-53; Generator.integers(0, n)
for n <= 2**32 = buffered 32-bit Lemire (low half of each raw draw first,
leftover half discarded at the end of the call).  Used by trainer.py:133-138
(seeds), envs/__init__.py:120-121 (starts) and buffer.py:136 (minibatch).
Pure-Python big-int arithmetic: small cases only.  Test infrastructure only.
"""

from __future__ import annotations

import numpy as np

MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1


def state_of(seed):
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def raw_stream(seed, count, skip=0):
    """`count` raw 64-bit outputs after skipping `skip` (state advanced first)."""
    s, inc = state_of(seed)
    for _ in range(skip):
        s = (s * MULT + inc) & MASK128
    out = []
    for _ in range(count):
        s = (s * MULT + inc) & MASK128
        hi, lo = s >> 64, s & MASK64
        rot = hi >> 58
        v = hi ^ lo
        out.append(((v >> rot) | (v << ((64 - rot) & 63))) & MASK64)
    return out


def uniform(seed, count):
    return np.array([(r >> 11) * 2.0 ** -53 for r in raw_stream(seed, count)])


def lemire_indices(raws, n, count):
    """Generator.integers(0, n, size=count) from a raw stream (n < 2**32)."""
    thresh = ((1 << 32) - n) % n
    out = []
    halves = []
    for r in raws:
        halves += [r & 0xFFFFFFFF, r >> 32]
    it = iter(halves)
    while len(out) < count:
        x = next(it)
        mprod = x * n
        if (mprod & 0xFFFFFFFF) < n:
            while (mprod & 0xFFFFFFFF) < thresh:
                x = next(it)
                mprod = x * n
        out.append(mprod >> 32)
    return np.array(out, dtype=np.int64)
