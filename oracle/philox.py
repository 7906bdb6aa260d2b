"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
1, 2, 3"), the counter-based generator that supplies the three uniforms a
guided sample draws (P:305 needs uniforms for the vMF
sampler).  Test infrastructure only -- see oracle/__init__.py.

Pinned by the published Random123 known-answer vectors
(tests/golden/philox4x32_10_kat.txt).
"""
import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """ctr: 4 arrays of uint32 values, key: 2 arrays (or scalars).

    Returns 4 uint64 arrays holding 32-bit outputs.  One round:
      (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
      c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    and the key is bumped by the Weyl constants between rounds.
    """
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK32 for c in ctr)
    k0 = np.asarray(key[0], dtype=np.uint64) & MASK32
    k1 = np.asarray(key[1], dtype=np.uint64) & MASK32
    for r in range(10):
        if r > 0:
            k0 = (k0 + np.uint64(W0)) & np.uint64(MASK32)
            k1 = (k1 + np.uint64(W1)) & np.uint64(MASK32)
        p0 = np.uint64(M0) * c0          # < 2^64, exact in uint64
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK32)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def sample_uniforms(n, seed, offset, count=3):
    """Uniforms for sample i (C-O11): key = (lo32(seed), hi32(seed)),
    counter = (lo32(i + offset), hi32(i + offset), 0, 0);
    u_j = (out_j >> 8) * 2^-24 for j = 0, 1, 2 (24-bit, in [0, 1)); count=4
    adds u_3 from out_3, the technique selector of combined sampling (C-A25).
    Returns float64 array [count, n]."""
    idx = np.arange(n, dtype=np.uint64) + np.uint64(offset)
    ctr = (idx & np.uint64(MASK32), idx >> np.uint64(32),
           np.zeros(n, np.uint64), np.zeros(n, np.uint64))
    key = (np.uint64(seed & MASK32), np.uint64((seed >> 32) & MASK32))
    o = philox4x32_10(ctr, key)
    return np.stack([(o[j] >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
                     for j in range(count)])
