"""Philox4x32-10 and the Gaussian test matrix G of each randUTV step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper draws ``G = randn(m - b(i-1), b)`` at step i (Fig.
fig:randUTV; also PAPER.md:632 §4.3 and the Theorem at).  It does
not name a generator.  Reading R2: a counter-based Philox4x32-10
(Salmon, Moraes, Dror, Shaw, SC'11) so that the CPU oracle and the GPU draw the
same numbers from (seed, step, row, column) without sharing state:

* key     = (lo32(seed), hi32(seed))
* counter = (p, c, step, purpose), p = row // 2, c = column, step = i - 1,
            purpose = 0 for the sketch.
* words x0..x3 -> two uniforms
        u  = (2 * (((x1 << 32) | x0) >> 12) + 1) * 2^-53
        u' = (2 * (((x3 << 32) | x2) >> 12) + 1) * 2^-53
  (52 random bits; exact in fp64; never 0 or 1).
* Box-Muller: rho = sqrt(-2 ln u), theta = 2 pi u';
        G[2p, c] = rho cos(theta),  G[2p+1, c] = rho sin(theta).

Pins: the round function against cuRAND's host-callable
``curand_Philox4x32_10`` (tests/test_oracle_philox.py), the integer->double
map by exact identities, the Gaussian by the Box-Muller identity and by
distribution tests.
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint32(0x9E3779B9)
PHILOX_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key) -> np.ndarray:
    """Ten Philox4x32 rounds.  ``ctr``: uint32 array of shape (4, N);
    ``key``: two uint32.  Returns the (4, N) uint32 output block.

    round:  (hi0, lo0) = M0 * c0;  (hi1, lo1) = M1 * c2   (32x32 -> 64 bit)
            c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    the key is bumped by (W0, W1) between rounds (9 bumps for 10 rounds).
    """
    c = [np.asarray(ctr[i], dtype=np.uint32).copy() for i in range(4)]
    k0 = np.uint32(key[0])
    k1 = np.uint32(key[1])
    for rnd in range(10):
        if rnd > 0:
            k0 = np.uint32((int(k0) + int(PHILOX_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(PHILOX_W1)) & 0xFFFFFFFF)
        p0 = PHILOX_M0 * c[0].astype(np.uint64)
        p1 = PHILOX_M1 * c[2].astype(np.uint64)
        hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
        lo0 = (p0 & _MASK32).astype(np.uint32)
        hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
        lo1 = (p1 & _MASK32).astype(np.uint32)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return np.stack(c)


def uniforms(words: np.ndarray):
    """Map a (4, N) Philox block to two arrays of uniforms in (0, 1)."""
    w01 = (words[1].astype(np.uint64) << np.uint64(32)) | words[0].astype(np.uint64)
    w23 = (words[3].astype(np.uint64) << np.uint64(32)) | words[2].astype(np.uint64)
    k01 = (w01 >> np.uint64(12)).astype(np.float64)  # < 2^52: exact
    k23 = (w23 >> np.uint64(12)).astype(np.float64)
    u = (2.0 * k01 + 1.0) * 2.0 ** -53
    u2 = (2.0 * k23 + 1.0) * 2.0 ** -53
    return u, u2


def seed_key(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return (seed & 0xFFFFFFFF, seed >> 32)


def gaussian_block(seed: int, step: int, rows: int, cols: int, purpose: int = 0) -> np.ndarray:
    """G (rows x cols, column-major float64) for randUTV step ``step`` (0-based,
    = i - 1 in the paper's 1-based loop)."""
    npairs = (rows + 1) // 2
    p = np.tile(np.arange(npairs, dtype=np.uint32), cols)
    c = np.repeat(np.arange(cols, dtype=np.uint32), npairs)
    ctr = np.stack([p, c, np.full_like(p, step), np.full_like(p, purpose)])
    u, u2 = uniforms(philox4x32_10(ctr, seed_key(seed)))
    rho = np.sqrt(-2.0 * np.log(u))
    theta = (2.0 * np.pi) * u2
    g = np.empty((2 * npairs, cols), dtype=np.float64, order="F")
    g[0::2, :] = (rho * np.cos(theta)).reshape(cols, npairs).T
    g[1::2, :] = (rho * np.sin(theta)).reshape(cols, npairs).T
    return np.asfortranarray(g[:rows, :])
