"""Philox4x32-10 (Salmon et al., SC'11), vectorised over numpy uint64 arrays.

TEST INFRASTRUCTURE (see oracle/__init__.py).

The paper draws its mask M_t, the atom permutation and the sample order "at
random" without naming a generator.  Reading R1 in
DESIGN.md: every random draw is a Philox4x32-10 block keyed by the 64-bit seed
(key = (seed mod 2^32, seed >> 32)) with a counter naming what is drawn, so the
oracle and the GPU produce identical draws.  Pinned against cuRAND's
``curand_Philox4x32_10`` compiled for the host (tests/test_oracle_rng.py).

Round function (per round, with key (k0, k1)):
    (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    k += (W0, W1)   between rounds
"""
import numpy as np

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Return the 4 output words for counters (c0, c1, c2, c3) under ``seed``.

    Inputs are broadcastable integer arrays holding values in [0, 2^32);
    outputs are four uint64 arrays holding uint32 values.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = int(seed) & 0xFFFFFFFF
    k1 = (int(seed) >> 32) & 0xFFFFFFFF
    m0 = np.uint64(PHILOX_M0)
    m1 = np.uint64(PHILOX_M1)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + PHILOX_W0) & 0xFFFFFFFF
            k1 = (k1 + PHILOX_W1) & 0xFFFFFFFF
        p0 = m0 * c0          # < 2^64: exact in uint64
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return c0, c1, c2, c3
