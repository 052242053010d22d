"""The blocked randUTV driver, step by step as in Fig. fig:randUTV.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md:919-989 (Fig. ``fig:randUTV``, §5.2) line by line, with the
readings of DESIGN.md §"Readings of the paper" (R1..R12):

    T = A; U = I_m; V = I_n
    for i = 1 : min(ceil(m/b), ceil(n/b))
      I1 = 1:b(i-1); I2 = b(i-1)+1 : min(bi, m); I3 = bi+1 : m
      J1, J2, J3 likewise over n
      if I3, J3 nonempty
        G = randn(m - b(i-1), b)                                      P:941 (R1, R2)
        Y = X^T G,  X = T([I2,I3],[J2,J3])
        repeat q: [Y <- orth(Y)]  Y = X^T (X Y)                       P:943-945 (+P:422-425, R5)
        [𝕍, ~] = qr(Y)                                                P:949 (Householder, R3/R4)
        T(:,[J2,J3]) = T(:,[J2,J3]) 𝕍 ;  V(:,[J2,J3]) = V(:,[J2,J3]) 𝕍   P:950-951 (all m rows, R6)
        [𝕌, R] = qr(T([I2,I3],J2))
        U(:,[I2,I3]) = U(:,[I2,I3]) 𝕌 ; T([I2,I3],J3) = 𝕌^T T([I2,I3],J3)
        T(I3,J2) = 0                                                  P:960 (exact zeros, R12)
        [Us, Ds, Vs] = svd(R(1:b,1:b))
        T(I2,J2) = Ds ; T(I2,J3) = Us^T T(I2,J3) ; U(:,I2) = U(:,I2) Us
        T(I1,J2) = T(I1,J2) Vs ; V(:,J2) = V(:,J2) Vs
        [early stop, R11]
      else
        economical SVD of T([I2,I3],[J2,J3]) (QR + small SVD if tall, R8)
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from .householder import apply_left_t, apply_right, geqr2, larft, thin_q, unit_lower
from .philox import gaussian_block
from .small_svd import small_svd


def randutv(A, b: int, q: int, seed: int, k_stop: int = 0, tol: float = 0.0,
            reortho: bool = True, build_ortho: bool = True, gaussian=None, record: bool = False, p: int = 0):
    """Factor A (m x n, m >= n) as U T V^T.

    Parameters follow the C-ABI ``randutv_factor`` (include/randutv.h):
    ``k_stop`` > 0 stops before the first step with b(i-1) >= k_stop;
    ``tol`` > 0 stops after a randomized step once ||T(I3,J3)||_F <= tol ||A||_F
    (reading R11); ``reortho`` re-orthonormalizes Y before every X Y (R5);
    ``build_ortho`` = False returns U = V = None (the paper's "no orthonormal
    matrices" mode).  ``gaussian(step, rows, cols)``
    overrides the Philox draw (tests only).  ``p`` > 0 over-samples the sketch
    (Remark remark:positivep; Fig. fig:stepUTVoversampling,
    PAPER.md:1754-1765): G gets b + p_i columns, p_i = min(p, n_i - b) (reading
    R23), and QR(Y) is replaced by QR of the b dominant left singular vectors of
    the extended Y.

    Returns a dict with U, T, V, k (columns processed), steps (randomized
    steps taken), trailing_fro = ||T(k+1:m, k+1:n)||_F and a_fro = ||A||_F.
    """
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    if b < 1 or q < 0 or k_stop < 0 or p < 0:
        raise ValueError("invalid b, q, k_stop or p")
    if not np.all(np.isfinite(A)):
        raise ValueError("non-finite input")
    if gaussian is None:
        def gaussian(step, rows, cols):
            return gaussian_block(seed, step, rows, cols)

    T = np.array(A, order="F", copy=True)
    U = np.eye(m, order="F") if build_ortho else None
    V = np.eye(n, order="F") if build_ortho else None
    a_fro = float(np.linalg.norm(A))
    s = min(math.ceil(m / b), math.ceil(n / b))
    steps, k_done = 0, 0
    log = []

    for i in range(1, s + 1):
        r0 = b * (i - 1)
        if k_stop > 0 and r0 >= k_stop:
            break
        e2 = min(b * i, m)   # end of I2 (exclusive, 0-based)
        f2 = min(b * i, n)   # end of J2
        I3_nonempty = b * i < m
        J3_nonempty = b * i < n
        if I3_nonempty and J3_nonempty:
            X = T[r0:, r0:]                                   # X = T([I2,I3],[J2,J3])
            p_i = min(p, (n - r0) - b)                        # R23 (p = 0: the paper's Fig. fig:randUTV)
            G = gaussian(i - 1, m - r0, b + p_i)              # P:941 (R1: m_i x b), P:1131 (m x (b+p))
            Y = X.T @ G
            for _ in range(q):
                if reortho:
                    Y = thin_q(Y)
                Y = X.T @ (X @ Y)
            if p_i > 0:                                       # [Z,~,~] = svd(Y,'econ')
                Z = scipy.linalg.svd(Y, full_matrices=False, lapack_driver="gesvd")[0]
                Y = np.asfortranarray(Z[:, :b])               # qr(Z(:,1:b))
            Fv, tau_v = geqr2(Y)
            Vv = unit_lower(Fv, b)
            Tv = larft(Vv, tau_v)
            T[:, r0:] = apply_right(T[:, r0:], Vv, Tv)        # P:950, all m rows (R6)
            if build_ortho:
                V[:, r0:] = apply_right(V[:, r0:], Vv, Tv)
            Fu, tau_u = geqr2(T[r0:, r0:f2])
            Vu = unit_lower(Fu, b)
            Tu = larft(Vu, tau_u)
            R = np.triu(Fu[:b, :b])
            if build_ortho:
                U[:, r0:] = apply_right(U[:, r0:], Vu, Tu)
            T[r0:, f2:] = apply_left_t(T[r0:, f2:], Vu, Tu)
            T[e2:, r0:f2] = 0.0
            T[r0:e2, r0:f2] = R
            Us, D, Vs = small_svd(R)
            T[r0:e2, r0:f2] = np.diag(D)
            T[r0:e2, f2:] = Us.T @ T[r0:e2, f2:]
            if build_ortho:
                U[:, r0:e2] = U[:, r0:e2] @ Us
            T[:r0, r0:f2] = T[:r0, r0:f2] @ Vs
            if build_ortho:
                V[:, r0:f2] = V[:, r0:f2] @ Vs
            steps += 1
            k_done = f2
            if record:
                log.append({"step": i, "G": G, "Y": Y, "Vv": Vv, "Tv": Tv, "Vu": Vu, "Tu": Tu,
                            "R": R, "D": D})
            if tol > 0 and np.linalg.norm(T[e2:, f2:]) <= tol * a_fro:
                break
        else:
            X = T[r0:, r0:]
            mi, ni = X.shape
            if mi < ni:                                       # fat: Remark "The case m < n"
                # unpivoted QR of the ROWS: X^T = Q [Rf; 0], Rf = Ur D Vr^T, so
                # X = Vr D (Q blockdiag(Ur, I))^T[:mi, :]: U_small = Vr and
                # V_small = Q blockdiag(Ur, I), a product of Householder reflectors
                Ff, tau_f = geqr2(X.T)
                Vf = unit_lower(Ff, mi)
                Tf = larft(Vf, tau_f)
                Ur, D, Vr = small_svd(np.triu(Ff[:mi, :mi]))
                if build_ortho:
                    U[:, r0:] = U[:, r0:] @ Vr
                    V[:, r0:] = apply_right(V[:, r0:], Vf, Tf)
                    V[:, r0:r0 + mi] = V[:, r0:r0 + mi] @ Ur
                T[:r0, r0:] = apply_right(T[:r0, r0:], Vf, Tf)
                T[:r0, r0:r0 + mi] = T[:r0, r0:r0 + mi] @ Ur
                T[r0:, r0:] = 0.0
                T[r0 + np.arange(mi), r0 + np.arange(mi)] = D
                k_done = m
                if record:
                    log.append({"step": i, "final": True, "D": D})
                break
            if mi > ni:                                       # tall: Remark rem:econ_svd
                Ff, tau_f = geqr2(X)
                Vf = unit_lower(Ff, ni)
                Tf = larft(Vf, tau_f)
                Us, D, Vs = small_svd(np.triu(Ff[:ni, :ni]))
                if build_ortho:
                    U[:, r0:] = apply_right(U[:, r0:], Vf, Tf)
                    U[:, r0:r0 + ni] = U[:, r0:r0 + ni] @ Us
            else:
                Us, D, Vs = small_svd(X)
                if build_ortho:
                    U[:, r0:] = U[:, r0:] @ Us
            if build_ortho:
                V[:, r0:] = V[:, r0:] @ Vs
            T[r0:, r0:] = 0.0
            T[r0 + np.arange(ni), r0 + np.arange(ni)] = D
            T[:r0, r0:] = T[:r0, r0:] @ Vs
            k_done = n
            if record:
                log.append({"step": i, "final": True, "D": D})
    trailing = float(np.linalg.norm(T[k_done:, k_done:])) if k_done < min(m, n) else 0.0
    out = {"U": U, "T": T, "V": V, "k": k_done, "steps": steps, "trailing_fro": trailing,
           "a_fro": a_fro}
    if record:
        out["log"] = log
    return out

