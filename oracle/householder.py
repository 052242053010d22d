"""Unpivoted Householder QR, compact-WY factor and its applications.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: §2.4 "Efficient factorizations of tall and thin matrices"
(PAPER.md:327-357): B = 𝕈 R with 𝕈 a product of b Householder reflectors,
stored in O(mb) words and applied with ~2mnb flops through the representation
𝕈 = I + W Y (Eq. eq:WYrepresentation; the references
[BiVL87, ScVL89, Joffrain 2006] at PAPER.md:351).  We use the equivalent
compact-WY form 𝕈 = H_1 H_2 ... H_k = I - V T V^T with V unit lower
trapezoidal and T upper triangular (W = -V T, Y = V^T).

Reading R3: the paper leaves the reflector sign open; we fix
LAPACK dlarfg's convention so that LAPACK's dgeqrf pins it:
    beta = -copysign(||x||_2, alpha),  tau = (beta - alpha) / beta,
    v = [1; x(2:) / (alpha - beta)];   if ||x(2:)|| == 0: tau = 0 (H = I).
"""
from __future__ import annotations

import math

import numpy as np


def house(x: np.ndarray):
    """Householder reflector of x (dlarfg).  Returns (v, tau, beta) with
    (I - tau v v^T) x = beta e_1 and v[0] = 1."""
    x = np.asarray(x, dtype=np.float64)
    alpha = float(x[0])
    xnorm = float(np.linalg.norm(x[1:])) if x.size > 1 else 0.0
    v = np.empty_like(x)
    v[0] = 1.0
    if xnorm == 0.0:
        v[1:] = x[1:]
        return v, 0.0, alpha
    beta = -math.copysign(math.hypot(alpha, xnorm), alpha)
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def geqr2(B: np.ndarray):
    """Unpivoted Householder QR of B (m x k), column by column (LAPACK dgeqr2).

    Returns (F, tau): F holds R on and above the diagonal and the reflector
    vectors (without their unit leading entry) below it.
    """
    F = np.array(B, dtype=np.float64, order="F", copy=True)
    m, k = F.shape
    kk = min(m, k)
    tau = np.zeros(kk)
    for j in range(kk):
        v, t, beta = house(F[j:, j])
        tau[j] = t
        F[j, j] = beta
        F[j + 1:, j] = v[1:]
        if t != 0.0 and j + 1 < k:
            w = F[j:, j + 1:].T @ v                 # w = C^T v
            F[j:, j + 1:] -= t * np.outer(v, w)     # C <- (I - tau v v^T) C
    return F, tau


def unit_lower(F: np.ndarray, k: int | None = None) -> np.ndarray:
    """The unit lower trapezoidal V (m x k) stored below the diagonal of F."""
    m = F.shape[0]
    k = min(F.shape) if k is None else k
    V = np.tril(F[:, :k], -1)
    V[np.arange(k), np.arange(k)] = 1.0
    return np.asfortranarray(V)


def larft(V: np.ndarray, tau: np.ndarray) -> np.ndarray:
    """Forward, column-wise T factor (LAPACK dlarft): H_1...H_k = I - V T V^T.

    T[i, i] = tau_i;  T[:i, i] = -tau_i T[:i, :i] (V[:, :i]^T v_i).
    """
    k = len(tau)
    T = np.zeros((k, k))
    for i in range(k):
        if tau[i] == 0.0:
            continue  # H_i = I: column i of T stays zero
        t = V[:, :i].T @ V[:, i]
        T[:i, i] = -tau[i] * (T[:i, :i] @ t)
        T[i, i] = tau[i]
    return T


def apply_right(C: np.ndarray, V: np.ndarray, T: np.ndarray) -> np.ndarray:
    """C 𝕈 = C (I - V T V^T) = C - (C V) T V^T."""
    return C - ((C @ V) @ T) @ V.T


def apply_left_t(C: np.ndarray, V: np.ndarray, T: np.ndarray) -> np.ndarray:
    """𝕈^T C = (I - V T^T V^T) C = C - V (T^T (V^T C))."""
    return C - V @ (T.T @ (V.T @ C))


def thin_q(Y: np.ndarray) -> np.ndarray:
    """Orthonormal basis of range(Y) as the first k columns of the Householder
    𝕈 of Y: Q1 = (I - V T V^T)[:, :k].  Used for the power-loop
    re-orthonormalization (reading R5)."""
    F, tau = geqr2(Y)
    k = len(tau)
    V = unit_lower(F, k)
    T = larft(V, tau)
    E = np.zeros((Y.shape[0], k))
    E[np.arange(k), np.arange(k)] = 1.0
    return np.asfortranarray(E - V @ (T @ V[:k, :].T))
