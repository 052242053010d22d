"""The b x b SVD of the active diagonal block.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:964 ``[U_small, D_small, V_small] = svd(R(1:b,1:b))`` and the final
block's ``svd`` at PAPER.md:971.  The paper calls a library SVD; so does the
oracle: LAPACK dgesvd through scipy (a library primitive used as one step).
Reading R9: D >= 0 non-increasing; singular-vector signs are free
(they change neither |diag T|, nor the rank-k errors at block boundaries, nor
any later step).  Canonical sign here: the largest-|.| entry of each V_small
column is positive (U_small follows).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def small_svd(R: np.ndarray):
    """R = Us diag(D) Vs^T with D non-increasing.  Returns (Us, D, Vs)."""
    U, s, Vh = scipy.linalg.svd(np.asarray(R, dtype=np.float64), full_matrices=True,
                                lapack_driver="gesvd")
    Vs = Vh.T.copy()
    k = len(s)
    idx = np.argmax(np.abs(Vs[:, :k]), axis=0)
    sgn = np.sign(Vs[idx, np.arange(k)])
    sgn[sgn == 0] = 1.0
    Vs[:, :k] *= sgn[None, :]
    U = U.copy()
    U[:, :k] *= sgn[None, :]
    return np.asfortranarray(U), s, np.asfortranarray(Vs)
