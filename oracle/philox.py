"""Philox4x32-10 counter-based generator, written out from its round definition.

Used for (a) the synthetic weights (weights are a pure function of a seed so
that the GPU side can generate them on-device with its own implementation of the same
generator), and (b) the Gumbel draws of stochastic verification (SURVEY amb. A9; SPEC S:43
"seeded, splittable per (session, round, purpose)").

Round (Salmon et al. 2011, Random123): with M0=0xD2511F53, M1=0xCD9E8D57,
  (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2
  c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  k <- (k0 + 0x9E3779B9, k1 + 0xBB67AE85)
ten rounds, the key bumped between rounds.  Pinned by the Random123 known-answer vectors
(tests/test_oracle_numerics.py).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised over broadcastable uint32-valued arrays; returns four uint64 arrays < 2**32."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK for c in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK
    k1 = np.asarray(k1, dtype=np.uint64) & MASK
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> S32, p0 & MASK
        hi1, lo1 = p1 >> S32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


def word(idx, c1, c2, c3, k0, k1):
    """The 32-bit word for element `idx` of a stream: counter (idx>>2, c1, c2, c3), word idx&3."""
    idx = np.asarray(idx, dtype=np.uint64)
    r = philox4x32_10(idx >> np.uint64(2), c1, c2, c3, k0, k1)
    sel = (idx & np.uint64(3)).astype(np.int64)
    out = np.where(sel == 0, r[0], np.where(sel == 1, r[1], np.where(sel == 2, r[2], r[3])))
    return out


def words_range(start: int, count: int, c1, c2, c3, k0, k1):
    """Words for elements start..start+count-1 (same values as `word`, 4x less work)."""
    if count <= 0:
        return np.zeros(0, np.uint64)
    g0 = start >> 2
    g1 = (start + count - 1) >> 2
    ctr = np.arange(g0, g1 + 1, dtype=np.uint64)
    r = philox4x32_10(ctr, c1, c2, c3, k0, k1)
    flat = np.stack(r, axis=1).reshape(-1)
    off = start - 4 * g0
    return flat[off:off + count]


def split_seed(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32
