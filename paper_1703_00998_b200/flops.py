"""Flop counts used for the GFLOP/s metric (measurement helper, not method arithmetic).

PAPER.md:1203-1207 (§5.4): randUTV without orthonormal matrices costs
    F_T(m, n, q) = (5 + 2q) m n^2 - (3 + 2q) n^3 / 3   flops.
SURVEY §8(d) / App. A.1: this is the continuum limit of the per-step sum
    sketch (2+4q) m_i n_i b + right apply 4 m n_i b + left apply 4 m_i (n_i - b) b,
used for early-stopped runs (config 5).  U/V formation (reported separately):
F_UV = (4 m^2 k - 4 m k^2 + 4 k^3/3) + (4 n^2 k - 4 n k^2 + 4 k^3/3), k = min(m, n).
"""
from __future__ import annotations

import math


def flops_T(m: int, n: int, q: int) -> float:
    return (5 + 2 * q) * m * n * n - (3 + 2 * q) * n ** 3 / 3.0


def flops_T_steps(m: int, n: int, b: int, q: int, k_stop: int = 0) -> float:
    tot = 0.0
    s = min(math.ceil(m / b), math.ceil(n / b))
    for i in range(1, s + 1):
        r0 = b * (i - 1)
        if k_stop > 0 and r0 >= k_stop:
            break
        if b * i < m and b * i < n:
            mi, ni = m - r0, n - r0
            tot += (2 + 4 * q) * mi * ni * b + 4 * m * ni * b + 4 * mi * (ni - b) * b
    return tot


def flops_UV(m: int, n: int) -> float:
    k = min(m, n)
    f = lambda r: 4.0 * r * r * k - 4.0 * r * k * k + 4.0 * k ** 3 / 3.0  # noqa: E731
    return f(m) + f(n)


def flops_cpqr(m: int, n: int) -> float:
    """Unpivoted QR / CPQR without Q."""
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
