"""Randomized SVD (Remark remark:RSVD) -- the NEXT row 3
workload built from the same steps as randUTV's sketch.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    G = randn(m, b + p)                          §3.3 step 1, Remark remark:oversampling
    Y = (A^T A)^q A^T G   [Y <- orth(Y) before every A Y, reading R5]   step 2
    Q = orth(Y)                                  step 3: Householder thin Q (R3)
    B = A Q                                      Remark RSVD (1)
    B = U D Vhat^T   (full SVD of the small B)  Remark RSVD (2), LAPACK gesvd
    V = Q Vhat                                   Remark RSVD (3)
and, with p > 0, the leading b singular triplets are kept (rank-b output).
The Gaussian is the step-0 draw of the randUTV Philox stream (reading R2).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from .householder import thin_q
from .philox import gaussian_block


def rsvd(A, b: int, q: int, seed: int, p: int = 0, reortho: bool = True):
    """Rank-b approximation A ~ U diag(D) V^T; returns (U m x b, D b, V n x b, Q n x (b+p))."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    if b < 1 or q < 0 or p < 0 or b + p > min(m, n):
        raise ValueError("need 1 <= b, 0 <= q, 0 <= p, b + p <= min(m, n)")
    G = gaussian_block(seed, 0, m, b + p)
    Y = A.T @ G
    for _ in range(q):
        if reortho:
            Y = thin_q(Y)
        Y = A.T @ (A @ Y)
    Q = thin_q(Y)
    B = A @ Q
    Ub, D, Vh = scipy.linalg.svd(B, full_matrices=False, lapack_driver="gesvd")
    V = Q @ Vh.T
    return np.asfortranarray(Ub[:, :b]), D[:b].copy(), np.asfortranarray(V[:, :b]), Q
