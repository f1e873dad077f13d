"""Philox4x32-10 counter-based generator (oracle side) — TEST INFRASTRUCTURE.

The paper draws C at random (Alg. 1 step 2; "generating a large number
of random numbers") but fixes no generator.  DESIGN.md §3.1 fixes
Philox4x32-10 (Salmon et al., SC'11, the Random123 reference) so that the CPU
oracle and the device path can replay the same C without sharing code.

Definition written out (vectorised over NumPy arrays of counters):
  per round:  (hi0, lo0) = M0 * c0 ;  (hi1, lo1) = M1 * c2   (32x32 -> 64)
              c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
              k = (k0 + W0, k1 + W1)      (bumped between rounds; 10 rounds)
Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt).
"""

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)
SHIFT32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Return (w0, w1, w2, w3) as uint64 arrays holding 32-bit words.

    c0..c3: counter words (scalars or broadcastable arrays, values < 2**32).
    k0, k1: key words (scalars).
    """
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    for rnd in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> SHIFT32, p0 & MASK32
        hi1, lo1 = p1 >> SHIFT32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if rnd < 9:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
    return c0, c1, c2, c3


def seed_key(seed):
    """Key words from a 64-bit seed: (seed & 0xffffffff, seed >> 32)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32
