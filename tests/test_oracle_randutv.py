"""Pins for the blocked oracle driver oracle/randutv.py.

Each pin is something other than the oracle itself:
* brute force: a dense transcription of the paper's *simplistic* algorithm
  (Fig. fig:randUTVmatlab) built on LAPACK complete QR and
  LAPACK SVD, fed the same G (the paper states the two algorithms are
  mathematically equivalent; reading R17);
* the Theorem of §5.3, exact identities for one step;
* textbook special cases (b >= n is an SVD; A = I; A = 0; exact rank b,
  PAPER.md:605-620 §4.2);
* invariants of any UTV factorization and Eckart-Young /
  interlacing inequalities.
"""
import math

import numpy as np
import pytest

import testmat
from oracle import gaussian_block, randutv
from oracle.small_svd import small_svd
from util import EPS, diag_blocks_ok, ek_fro, invariants


# ----------------------------------------------------------------------------- brute force
def simplistic_randutv(A, b, q, seed, reortho=True, p=0):
    """Fig. fig:randUTVmatlab with dense unitary matrices (O(n^4)); stepUTV's
    ``svd(A*V(:,1:b))`` realised as QR + small SVD (Remark rem:econ_svd).
    p > 0: stepUTV of Fig. fig:stepUTVoversampling,
    ``[Z,~,~] = svd(Y,'econ'); [V,~] = qr(Z(:,1:b))`` with numpy's SVD (LAPACK
    gesdd, not the oracle's gesvd), p_i = min(p, n_i - b) (reading R23)."""
    m, n = A.shape
    T = A.copy(); U = np.eye(m); V = np.eye(n)
    for i in range(1, math.ceil(min(m, n) / b) + 1):
        r0 = b * (i - 1)
        Ai = T[r0:, r0:]
        if Ai.shape[0] > b and Ai.shape[1] > b:
            p_i = min(p, Ai.shape[1] - b)
            G = gaussian_block(seed, i - 1, Ai.shape[0], b + p_i)
            Y = Ai.T @ G
            for _ in range(q):
                if reortho:
                    Y = np.linalg.qr(Y)[0]
                Y = Ai.T @ (Ai @ Y)
            if p_i > 0:
                Y = np.linalg.svd(Y, full_matrices=False)[0][:, :b]
            VV = np.linalg.qr(Y, mode="complete")[0]
            UU, R = np.linalg.qr(Ai @ VV[:, :b], mode="complete")
            Us, D, W = small_svd(R[:b, :b])
            UU[:, :b] = UU[:, :b] @ Us
            TT = np.zeros_like(Ai)
            TT[:b, :b] = np.diag(D)
            TT[:, b:] = UU.T @ Ai @ VV[:, b:]
            TT[b:, :b] = 0.0
            VV[:, :b] = VV[:, :b] @ W
        else:
            UU, s, Vh = np.linalg.svd(Ai, full_matrices=True)
            VV = Vh.T.copy()
            k = len(s)                                      # same canonical sign as small_svd
            sg = np.sign(VV[np.argmax(np.abs(VV[:, :k]), axis=0), np.arange(k)])
            VV[:, :k] *= sg[None, :]
            UU[:, :k] *= sg[None, :]
            TT = np.zeros_like(Ai)
            TT[np.arange(len(s)), np.arange(len(s))] = s
        U[:, r0:] = U[:, r0:] @ UU
        V[:, r0:] = V[:, r0:] @ VV
        T[r0:, r0:] = TT
        T[:r0, r0:] = T[:r0, r0:] @ VV
    return U, T, V


@pytest.mark.parametrize("m,n,b,q", [(48, 48, 8, 1), (60, 45, 8, 2), (40, 33, 10, 0)])
def test_efficient_equals_simplistic(m, n, b, q):
    A = testmat.gaussian(m, n, seed=m + n)
    r = randutv(A, b, q, seed=9)
    U2, T2, V2 = simplistic_randutv(A, b, q, seed=9)
    a = np.linalg.norm(A)
    np.testing.assert_allclose(np.abs(np.diag(r["T"])), np.abs(np.diag(T2)), rtol=1e-10, atol=1e-13 * a)
    np.testing.assert_allclose(ek_fro(r["T"]), ek_fro(T2), rtol=1e-10, atol=1e-13 * a)
    # with the shared canonical SVD sign the factors agree entry by entry
    np.testing.assert_allclose(r["T"], T2, atol=1e-11 * a)
    np.testing.assert_allclose(r["U"], U2, atol=1e-10)
    np.testing.assert_allclose(r["V"], V2, atol=1e-10)


@pytest.mark.parametrize("m,n,b,q", [(33, 48, 8, 1), (20, 50, 8, 2), (40, 41, 10, 0), (16, 40, 8, 1)])
def test_fat_efficient_equals_simplistic(m, n, b, q):
    """m < n (Remark "The case m < n"): the final fat block by a QR of
    its rows; the dense transcription takes a full LAPACK SVD of that block."""
    A = testmat.gaussian(m, n, seed=m * n)
    r = randutv(A, b, q, seed=4)
    U2, T2, V2 = simplistic_randutv(A, b, q, seed=4)
    a = np.linalg.norm(A)
    np.testing.assert_allclose(np.abs(np.diag(r["T"])), np.abs(np.diag(T2)), rtol=1e-10, atol=1e-13 * a)
    np.testing.assert_allclose(ek_fro(r["T"]), ek_fro(T2), rtol=1e-10, atol=1e-13 * a)
    inv = invariants(A, r["U"], r["T"], r["V"])
    assert inv["recon"] < 1e-14 * n and inv["orth_u"] < 1e-13 * n and inv["orth_v"] < 1e-13 * n
    assert inv["tril_max"] == 0.0 and r["k"] == m


def test_fat_b_geq_m_is_svd():
    """b >= m: a single final step = the SVD of A (textbook), T = [diag(sigma) 0]."""
    A = testmat.gaussian(12, 30, 8)
    r = randutv(A, b=16, q=1, seed=0)
    T = r["T"]
    np.testing.assert_allclose(np.diag(T), np.linalg.svd(A, compute_uv=False), rtol=1e-13)
    off = T.copy(); off[np.arange(12), np.arange(12)] = 0
    assert np.all(off == 0)
    inv = invariants(A, r["U"], T, r["V"])
    assert inv["recon"] < 1e-14 * 30 and inv["orth_v"] < 1e-13 * 30


@pytest.mark.parametrize("m,n,b,q,p", [(48, 48, 8, 1, 5), (60, 45, 8, 2, 8), (40, 33, 10, 0, 3)])
def test_oversampling_efficient_equals_simplistic(m, n, b, q, p):
    """Over-sampled randUTV (Remark remark:positivep) vs the dense transcription
    of Fig. fig:stepUTVoversampling: Z's column signs are free (LAPACK gesvd vs
    gesdd), which flips signs of T's rows/columns but not |diag T| nor e_k."""
    A = testmat.gaussian(m, n, seed=m + n + p)
    r = randutv(A, b, q, seed=9, p=p)
    U2, T2, V2 = simplistic_randutv(A, b, q, seed=9, p=p)
    a = np.linalg.norm(A)
    np.testing.assert_allclose(np.abs(np.diag(r["T"])), np.abs(np.diag(T2)), rtol=1e-10, atol=1e-13 * a)
    np.testing.assert_allclose(ek_fro(r["T"]), ek_fro(T2), rtol=1e-10, atol=1e-13 * a)
    np.testing.assert_allclose(np.abs(r["T"]), np.abs(T2), atol=1e-11 * a)
    inv = invariants(A, r["U"], r["T"], r["V"])
    assert inv["recon"] < 1e-14 * n and inv["orth_u"] < 1e-13 * n and inv["orth_v"] < 1e-13 * n
    # p = 0 is the paper's Fig. fig:randUTV exactly
    r0 = randutv(A, b, q, seed=9, p=0)
    r1 = randutv(A, b, q, seed=9)
    assert np.array_equal(r0["T"], r1["T"])


def test_oversampling_improves_first_block():
    """Remark remark:positivep / App. app:oversampling: over-sampling aligns
    col(V_1) better with the dominant right singular vectors, so the first
    block's D (= sigma(A V_1) <= sigma_j, interlacing) moves towards sigma."""
    m = n = 200
    b = 20
    rng = np.random.default_rng(5)
    s = 0.95 ** np.arange(n)
    A = (np.linalg.qr(rng.standard_normal((m, n)))[0] * s) @ np.linalg.qr(rng.standard_normal((n, n)))[0].T
    gaps = []
    for p in (0, 10):
        d = np.mean([np.sum(s[:b] - np.diag(randutv(A, b, 0, seed=t, k_stop=b, p=p, build_ortho=False)["T"])[:b])
                     for t in range(6)])
        gaps.append(d)
    assert gaps[1] < gaps[0]


# ----------------------------------------------------------------------------- Theorem §5.3
@pytest.mark.parametrize("q", [0, 1, 2])
def test_theorem_5_3_identities(q):
    m, n, b = 300, 200, 20
    rng = np.random.default_rng(3)
    s = 0.9 ** np.arange(n)
    A = (np.linalg.qr(rng.standard_normal((m, n)))[0] * s) @ np.linalg.qr(rng.standard_normal((n, n)))[0].T
    r = randutv(A, b, q, seed=1, k_stop=b)                 # exactly one step
    T = r["T"]
    G = gaussian_block(1, 0, m, b)
    Y = A.T @ G
    for _ in range(q):
        Y = np.linalg.qr(Y)[0]                              # same span, LAPACK (not the oracle's QR)
        Y = A.T @ (A @ Y)
    Q = np.linalg.qr(Y)[0]
    W = np.linalg.qr(A @ Y)[0]
    for ordv in (2, "fro"):
        lhs_a = np.linalg.norm(A - A @ Q @ Q.T, ordv)
        rhs_a = np.linalg.norm(T[:, b:], ordv)              # ||[T12; T22]||
        assert abs(lhs_a - rhs_a) <= 1e-13 * s[0]
        lhs_b = np.linalg.norm(A - W @ (W.T @ A), ordv)
        rhs_b = np.linalg.norm(T[b:, b:], ordv)             # ||T22||
        assert abs(lhs_b - rhs_b) <= 1e-11 * s[0]
    # first block D = svd(A Q) exactly (library re-derivation from the same G)
    np.testing.assert_allclose(np.diag(T)[:b], np.linalg.svd(A @ Q, compute_uv=False), rtol=1e-12)


# ----------------------------------------------------------------------------- special cases
@pytest.mark.parametrize("m,n", [(30, 30), (50, 20)])
def test_b_geq_n_is_svd(m, n):
    A = testmat.gaussian(m, n, 4)
    r = randutv(A, b=max(m, n), q=1, seed=0)
    d = np.diag(r["T"])
    np.testing.assert_allclose(d, np.linalg.svd(A, compute_uv=False), rtol=1e-13)
    off = r["T"].copy(); off[np.arange(n), np.arange(n)] = 0
    assert np.all(off == 0)
    inv = invariants(A, r["U"], r["T"], r["V"])
    assert inv["recon"] < 1e-14 * n


def test_identity_and_zero():
    n, b = 40, 8
    r = randutv(np.eye(n), b, 1, 0)
    np.testing.assert_allclose(r["T"], np.eye(n), atol=1e-13)
    r = randutv(np.zeros((n, n)), b, 1, 0)
    assert np.all(r["T"] == 0)
    assert np.linalg.norm(r["U"].T @ r["U"] - np.eye(n)) < 1e-13
    assert np.linalg.norm(r["V"].T @ r["V"] - np.eye(n)) < 1e-13


def test_exact_rank_b_ideal_case():
    """rank(A) = b: the first step finds the dominant subspaces exactly, so
    T12 = 0 and T22 = 0 to rounding."""
    rng = np.random.default_rng(8)
    m, n, b = 120, 90, 10
    A = rng.standard_normal((m, b)) @ rng.standard_normal((b, n))
    r = randutv(A, b, 1, 5, k_stop=b)
    T = r["T"]
    a = np.linalg.norm(A)
    assert np.linalg.norm(T[:b, b:]) <= 1e-12 * a
    assert np.linalg.norm(T[b:, b:]) <= 1e-12 * a
    np.testing.assert_allclose(np.diag(T)[:b], np.linalg.svd(A, compute_uv=False)[:b], rtol=1e-12)


# ----------------------------------------------------------------------------- invariants
CASES = [
    ("c1", dict(scale=1.0)),             # 500 x 500, b=50, q=1: BASELINE config 1 itself
    ("c2", dict(scale=0.1)),             # 300 x 300 exponential decay, b=75 -> reduced
    ("c3", dict(scale=0.05)),            # 500 x 500 S-shape, b=62
    ("c4", dict(scale=0.02)),            # 400 x 160 tall Gaussian, b=20: tall final block
]


@pytest.mark.parametrize("name,kw", CASES)
def test_invariants(name, kw):
    c = testmat.config(name, **kw)
    A = c.A
    m, n = A.shape
    r = randutv(A, c.b, c.q, c.seed)
    U, T, V = r["U"], r["T"], r["V"]
    inv = invariants(A, U, T, V)
    assert inv["recon"] <= 1e-13 * n
    assert inv["orth_u"] <= 1e-13 * n and inv["orth_v"] <= 1e-13 * n
    assert inv["tril_max"] == 0.0                          # exact triangularity
    assert inv["fro_rel"] <= n * EPS
    assert r["k"] == n
    assert diag_blocks_ok(T, c.b, n)
    sv = np.linalg.svd(A, compute_uv=False)
    d = np.diag(T)
    assert np.all(d[: c.b] <= sv[: c.b] * (1 + 1e-12))     # Cauchy interlacing, first block
    ek = ek_fro(T)
    tail = np.sqrt(np.concatenate([np.cumsum((sv ** 2)[::-1])[::-1], [0.0]]))
    assert np.all(ek >= tail * (1 - 1e-10) - 1e-14 * np.linalg.norm(A))   # Eckart-Young floor
    if m == n:                                             # |det| identity
        big = sv > 1e-6 * sv[0]
        if big.all():
            assert abs(np.sum(np.log(d)) - np.sum(np.log(sv))) < 1e-8 * n


def test_known_spectrum_band():
    """|diag T| tracks the known sigma (PAPER.md:1562-1587 prose; figure missing):
    a loose band on entries above the rounding floor."""
    c = testmat.config("c2", scale=0.15)       # 450 x 450, b=112
    r = randutv(c.A, c.b, 2, c.seed, build_ortho=False)
    d, s = np.diag(r["T"]), c.sigma
    sel = s > 1e-10
    ratio = d[sel] / s[sel]
    assert ratio.min() > 0.5 and ratio.max() < 2.0


def test_ragged_final_block():
    A = testmat.gaussian(150, 150, 2)
    r = randutv(A, 32, 1, 3)                                # final block 22 x 22
    inv = invariants(A, r["U"], r["T"], r["V"])
    assert inv["recon"] < 1e-13 * 150 and inv["tril_max"] == 0
    assert diag_blocks_ok(r["T"], 32, 150)


# ----------------------------------------------------------------------------- early stop
def test_k_stop_and_tol():
    n, rank = 200, 30
    c = testmat.Case("lr", testmat.low_rank_plus_noise(n, rank, 1e-8, 3), 16, 1, 3)
    r = randutv(c.A, 16, 1, 3, k_stop=40)                  # rounds up to 48
    assert r["k"] == 48 and r["steps"] == 3
    T = r["T"]
    assert np.all(T[48:, :48] == 0)
    assert abs(r["trailing_fro"] - np.linalg.norm(T[48:, 48:])) <= 1e-15 * r["a_fro"]
    inv = invariants(c.A, r["U"], T, r["V"])
    assert inv["recon"] < 1e-13 * n
    # tolerance stop: after the step that crosses the rank the trailing norm is noise-level
    r2 = randutv(c.A, 16, 1, 3, tol=1e-6)
    assert r2["k"] == 32 and r2["trailing_fro"] <= 1e-6 * r2["a_fro"]
    noise = 1e-8 * math.sqrt((n - 32) * (n - 32))
    assert r2["trailing_fro"] < 5 * noise


def test_reortho_invariance_and_determinism():
    A = testmat.gaussian(120, 120, 6)
    r1 = randutv(A, 16, 2, 1, build_ortho=False, reortho=True)
    r2 = randutv(A, 16, 2, 1, build_ortho=False, reortho=False)
    np.testing.assert_allclose(np.diag(r1["T"]), np.diag(r2["T"]), rtol=1e-11)
    r3 = randutv(A, 16, 2, 1, build_ortho=False, reortho=True)
    assert np.array_equal(r1["T"], r3["T"])


def test_errors():
    with pytest.raises(ValueError):
        randutv(np.ones((3, 5)), 0, 1, 0)
    with pytest.raises(ValueError):
        randutv(np.full((4, 4), np.nan), 2, 1, 0)
    with pytest.raises(ValueError):
        randutv(np.ones((4, 4)), 0, 1, 0)
