"""Pins for oracle/householder.py (§2.4; reading R3)."""
import json
import os

import numpy as np
import scipy.linalg.lapack as lapack

from oracle import householder as hh

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_closed_form_3_4():
    g = json.load(open(os.path.join(GOLD, "householder_3_4.json")))
    v, tau, beta = hh.house(np.array(g["x"]))
    assert beta == g["beta"] and abs(tau - g["tau"]) < 1e-15
    np.testing.assert_allclose(v, g["v"], rtol=0, atol=1e-16)
    H = np.eye(2) - tau * np.outer(v, v)
    np.testing.assert_allclose(H, g["H"], atol=1e-15)
    np.testing.assert_allclose(H @ g["x"], [g["beta"], 0.0], atol=1e-14)


def test_sign_conventions():
    # alpha = 0 -> sign(0) = + -> beta = -||x||
    v, tau, beta = hh.house(np.array([0.0, 2.0]))
    assert beta == -2.0 and tau == 1.0
    # negative alpha -> positive beta
    v, tau, beta = hh.house(np.array([-3.0, 4.0]))
    assert beta == 5.0
    # nothing below the diagonal -> H = I, tau = 0, beta = alpha (also for alpha < 0)
    v, tau, beta = hh.house(np.array([-7.0, 0.0, 0.0]))
    assert tau == 0.0 and beta == -7.0


def test_geqr2_matches_lapack_dgeqrf():
    """Library pin: LAPACK dgeqrf produces the same reflectors and tau (dlarfg convention)."""
    rng = np.random.default_rng(1)
    for (m, k) in [(50, 8), (37, 37), (200, 30), (9, 1)]:
        B = rng.standard_normal((m, k))
        F, tau = hh.geqr2(B)
        qr, tau_l, _, info = lapack.dgeqrf(np.asfortranarray(B))
        assert info == 0
        np.testing.assert_allclose(F, qr, rtol=0, atol=1e-12 * np.abs(qr).max())
        np.testing.assert_allclose(tau, tau_l, rtol=0, atol=1e-13)


def test_larft_equals_explicit_product():
    """I - V T V^T equals H_1 H_2 ... H_k formed explicitly."""
    rng = np.random.default_rng(2)
    m, k = 40, 6
    F, tau = hh.geqr2(rng.standard_normal((m, k)))
    V = hh.unit_lower(F)
    T = hh.larft(V, tau)
    Q = np.eye(m)
    for j in range(k):
        Q = Q @ (np.eye(m) - tau[j] * np.outer(V[:, j], V[:, j]))
    np.testing.assert_allclose(np.eye(m) - V @ T @ V.T, Q, atol=1e-13 * np.sqrt(m))
    assert np.allclose(np.tril(T, -1), 0)


def test_larft_with_identity_reflector():
    """tau = 0 columns (H = I) give zero T columns; product still exact."""
    B = np.zeros((6, 3)); B[:, 0] = [1, 2, 3, 4, 5, 6]; B[:, 2] = [0, 1, 0, 0, 0, 1]
    F, tau = hh.geqr2(B)
    assert tau[1] == 0.0
    V = hh.unit_lower(F); T = hh.larft(V, tau)
    assert np.all(T[:, 1] == 0)
    Q = np.eye(6) - V @ T @ V.T
    R = np.triu(F[:3, :3])
    np.testing.assert_allclose(Q[:, :3] @ R, B, atol=1e-14)


def test_reconstruction_orthogonality_and_applications():
    rng = np.random.default_rng(3)
    m, k, n = 120, 16, 30
    B = rng.standard_normal((m, k))
    F, tau = hh.geqr2(B)
    V = hh.unit_lower(F); T = hh.larft(V, tau)
    Q = np.eye(m) - V @ T @ V.T
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) < 1e-13 * np.sqrt(m)
    R = np.zeros((m, k)); R[:k] = np.triu(F[:k])
    assert np.linalg.norm(B - Q @ R) < 1e-13 * np.linalg.norm(B)
    C = rng.standard_normal((n, m))
    np.testing.assert_allclose(hh.apply_right(C, V, T), C @ Q, atol=1e-13 * np.linalg.norm(C))
    C2 = rng.standard_normal((m, n))
    np.testing.assert_allclose(hh.apply_left_t(C2, V, T), Q.T @ C2, atol=1e-13 * np.linalg.norm(C2))
    Q1 = hh.thin_q(B)
    np.testing.assert_allclose(Q1, Q[:, :k], atol=1e-14)
    # Q1 spans range(B): B = Q1 R1 with R1 = Q1^T B upper triangular
    np.testing.assert_allclose(np.tril(Q1.T @ B, -1), 0, atol=1e-12)


def test_triangular_rebasis_invariance():
    """Householder Q(Y M) = Q(Y) for upper-triangular M (basis of reading R5)."""
    rng = np.random.default_rng(4)
    Y = rng.standard_normal((80, 10))
    M = np.triu(rng.standard_normal((10, 10))) + 5 * np.eye(10)
    M[3, 3] *= -1  # negative diagonal entries only flip reflector-free signs
    F1, t1 = hh.geqr2(Y)
    F2, t2 = hh.geqr2(Y @ M)
    np.testing.assert_allclose(hh.unit_lower(F1), hh.unit_lower(F2), atol=1e-12)
    np.testing.assert_allclose(t1, t2, atol=1e-13)
