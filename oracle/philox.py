"""Philox4x32-10 counter-based RNG + Box-Muller (TEST INFRASTRUCTURE; see oracle/__init__.py).

The paper draws "randomly generated" vectors for the block expansion (Alg. 3 line 8,
PAPER.md:407) and a cold start block but names no generator (DESIGN.md
reading R11). Both sides implement the same counter-based generator, so the oracle and
the CUDA path draw identical streams without sharing code:

  Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3"):
    round:  (hi0,lo0) = mulhilo(M0, c0); (hi1,lo1) = mulhilo(M1, c2)
            c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    key bump between rounds: k0 += W0, k1 += W1;  10 rounds.
  Matrix entry E[i, j] of an n x q block (column-major linear index l = i + j*n):
    counter = (l >> 1, stream, ctx, tag), key = (seed_lo, seed_hi)
    u1 = ((x0 >> 5) * 2^26 + (x1 >> 6) + 0.5) * 2^-53,  u2 likewise from (x2, x3)
    l even -> sqrt(-2 ln u1) cos(2 pi u2);  l odd -> sqrt(-2 ln u1) sin(2 pi u2)
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint32 arrays (broadcast). Returns 4 uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = (x.copy() for x in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for r in range(10):
            p0 = M0 * c0.astype(np.uint64)
            p1 = M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            if r < 9:
                k0 = np.uint32(k0 + W0)
                k1 = np.uint32(k1 + W1)
    return c0, c1, c2, c3


def _u53(a, b):
    return ((a >> np.uint32(5)).astype(np.float64) * 67108864.0
            + (b >> np.uint32(6)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def gaussian_block(n, q, seed, stream, ctx=0, tag=0):
    """n x q standard-normal block (column-major semantics), per the mapping above."""
    total = n * q
    l = np.arange(total, dtype=np.uint64)
    half = (l >> np.uint64(1)).astype(np.uint32)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    x0, x1, x2, x3 = philox4x32_10(half, np.uint32(stream & 0xFFFFFFFF),
                                   np.uint32(ctx & 0xFFFFFFFF), np.uint32(tag & 0xFFFFFFFF),
                                   seed & 0xFFFFFFFF, seed >> 32)
    u1 = _u53(x0, x1)
    u2 = _u53(x2, x3)
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    odd = (l & np.uint64(1)).astype(bool)
    z = np.where(odd, rad * np.sin(ang), rad * np.cos(ang))
    return z.reshape((q, n)).T.copy()
