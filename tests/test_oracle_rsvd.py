"""Pins of the RSVD oracle (Remark remark:RSVD)."""
import numpy as np
import pytest

import testmat
from oracle import gaussian_block, rsvd
from util import EPS


def test_error_identity_and_small_svd():
    """E = A - A Q Q^T = A - U D V^T exactly for p = 0, and D =
    sigma(A Q) with Q re-derived by LAPACK from the same G."""
    m, n, b, q = 300, 200, 20, 1
    rng = np.random.default_rng(2)
    s = 0.9 ** np.arange(n)
    A = (np.linalg.qr(rng.standard_normal((m, n)))[0] * s) @ np.linalg.qr(rng.standard_normal((n, n)))[0].T
    U, D, V, Q = rsvd(A, b, q, seed=3)
    Y = A.T @ gaussian_block(3, 0, m, b)
    for _ in range(q):
        Y = np.linalg.qr(Y)[0]
        Y = A.T @ (A @ Y)
    Ql = np.linalg.qr(Y)[0]                                  # LAPACK, same span
    e1 = np.linalg.norm(A - A @ Ql @ Ql.T)
    e2 = np.linalg.norm(A - (U * D) @ V.T)
    assert abs(e1 - e2) <= 1e-13 * s[0] * n
    np.testing.assert_allclose(D, np.linalg.svd(A @ Ql, compute_uv=False), rtol=1e-12)
    assert np.linalg.norm(U.T @ U - np.eye(b)) < 1e-13 * m and np.linalg.norm(V.T @ V - np.eye(b)) < 1e-13 * n


def test_exact_rank_recovery_and_eckart_young():
    A = testmat.gaussian(120, 8, 1) @ testmat.gaussian(8, 90, 2)       # rank 8
    U, D, V, _ = rsvd(A, 8, 1, seed=0)
    assert np.linalg.norm(A - (U * D) @ V.T) <= 1e-12 * np.linalg.norm(A)
    np.testing.assert_allclose(D, np.linalg.svd(A, compute_uv=False)[:8], rtol=1e-12)
    B = testmat.gaussian(150, 100, 5)
    sv = np.linalg.svd(B, compute_uv=False)
    for p in (0, 10):
        U, D, V, _ = rsvd(B, 10, 2, seed=1, p=p)
        err = np.linalg.norm(B - (U * D) @ V.T)
        assert err >= np.sqrt(np.sum(sv[10:] ** 2)) * (1 - 1e-12)      # Eckart-Young floor
        assert np.all(D <= sv[:10] * (1 + 1e-12))                      # interlacing


def test_arguments():
    with pytest.raises(ValueError):
        rsvd(np.ones((5, 4)), 3, 1, 0, p=2)
