"""Philox4x32-10 counter-based RNG and the stream layout (ORACLE — test infrastructure only).

Algorithm: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3"
(SC'11), Philox4x32 with R=10 rounds: per round
    (hi0, lo0) = mulhilo(M0, c0); (hi1, lo1) = mulhilo(M1, c2)
    c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
then the key is bumped by the Weyl constants (W0, W1) before the next round.

The paper only says regrowth is "random" (Alg. 2) and the
initial graph is Erdos-Renyi; a counter-based generator lets
every replica (and this oracle) draw the same numbers without communication
(BASELINE.json north_star: "Evolution uses counter-based RNG so all ranks agree
without broadcast").  The stream layout below is this build's own spec
(SURVEY.md §8(c) O11):

    key     = (seed & 0xffffffff, seed >> 32)
    counter = (idx & 0xffffffff, idx >> 32, purpose << 24 | rank << 16 | layer, c3)

    purpose 1 INIT candidates      idx = m (candidate number)        c3 = 0
    purpose 2 INIT dense values    idx = i * n_out + j               c3 = 0
    purpose 3 REGROW candidates    idx = m                           c3 = evolve index e
    purpose 4 DROPOUT              idx = j * 2^32 + (b >> 2)         c3 = global step (low 32 bits)
                                   word = b & 3
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)

PURPOSE_INIT = 1
PURPOSE_INIT_DENSE = 2
PURPOSE_REGROW = 3
PURPOSE_DROPOUT = 4


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10.  c0..c3: uint32-valued arrays (or scalars); k0, k1: ints.
    Returns four uint32 arrays."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        p0 = M0 * c0                 # < 2^64, exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0)
        if r < 9:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


def stream(seed: int, purpose: int, rank: int, layer: int, c3: int, idx):
    """The four 32-bit words for stream positions ``idx`` (uint64 array) of one stream."""
    idx = np.asarray(idx, dtype=np.uint64)
    lo = idx & MASK32
    hi = idx >> np.uint64(32)
    c2 = ((purpose & 0xFF) << 24) | ((rank & 0xFF) << 16) | (layer & 0xFFFF)
    return philox4x32_10(lo, hi, np.uint64(c2), np.uint64(c3 & 0xFFFFFFFF),
                         seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
