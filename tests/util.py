"""Test-side measures of a UTV factorization (never used by the product)."""
import numpy as np

EPS = np.finfo(np.float64).eps


def ek_fro(T: np.ndarray) -> np.ndarray:
    """e_k^F = ||A - U(:,1:k) T(1:k,:) V^T||_F = ||T(k+1:m, :)||_F for k = 0..n
    (exact for orthogonal U, V; PAPER.md:1441-1455 and SURVEY §8(c) item 18)."""
    r2 = np.sum(np.asarray(T) ** 2, axis=1)
    tail = np.concatenate([np.cumsum(r2[::-1])[::-1], [0.0]])
    n = T.shape[1]
    return np.sqrt(tail[: n + 1])


def parity_floor(n: int, a_fro: float, c: float = 1.0) -> float:
    """Absolute rounding floor F = c n eps ||A||_F of the parity rule (R18)."""
    return c * n * EPS * a_fro


def check_parity(T_test, T_ref, a_fro, rtol_diag=1e-10, rtol_ek=1e-8, c=1.0):
    """|diag T| within rtol_diag relative + F; e_k^F within rtol_ek relative + F."""
    n = T_ref.shape[1]
    F = parity_floor(max(T_ref.shape), a_fro, c)
    dt, dr = np.abs(np.diag(T_test)), np.abs(np.diag(T_ref))
    bad_d = np.abs(dt - dr) > rtol_diag * dr + F
    et, er = ek_fro(T_test), ek_fro(T_ref)
    bad_e = np.abs(et - er) > rtol_ek * er + F
    return {
        "diag_ok": not bad_d.any(), "ek_ok": not bad_e.any(),
        "diag_max_rel": float(np.max(np.abs(dt - dr) / np.maximum(dr, F))),
        "ek_max_rel": float(np.max(np.abs(et - er) / np.maximum(er, F))),
        "n_bad_diag": int(bad_d.sum()), "n_bad_ek": int(bad_e.sum()),
    }


def invariants(A, U, T, V):
    A = np.asarray(A); m, n = A.shape
    out = {"tril_max": float(np.max(np.abs(np.tril(T, -1)))) if min(m, n) > 1 else 0.0,
           "fro_rel": abs(np.linalg.norm(T) - np.linalg.norm(A)) / max(np.linalg.norm(A), 1e-300)}
    if U is not None:
        out["recon"] = float(np.linalg.norm(A - U @ T @ V.T) / max(np.linalg.norm(A), 1e-300))
        out["orth_u"] = float(np.linalg.norm(U.T @ U - np.eye(m)))
        out["orth_v"] = float(np.linalg.norm(V.T @ V - np.eye(n)))
    return out


def diag_blocks_ok(T, b, k):
    """Each processed b x b diagonal block is diagonal with non-negative,
    non-increasing entries."""
    for r0 in range(0, k, b):
        e = min(r0 + b, k)
        blk = T[r0:e, r0:e]
        d = np.diag(blk)
        if np.any(blk - np.diag(d)):
            return False
        if np.any(d < 0) or np.any(np.diff(d) > 0):
            return False
    return True


def selection_well_posed(A, b, q, seed, p, ref, k_stop=0):
    """Over-sampling (R23): Z = the b dominant left singular
    vectors of the (b + p_i)-column sketch is determined only when
    sigma_b(Y') and sigma_{b+1}(Y') are separated; on flat trailing spectra
    (e.g. Gaussian inputs after some steps) it is not, and any rounding
    difference selects a different, equally valid subspace.  Detected from the
    oracle itself: re-run it on A perturbed by 1e-15 relative noise; if its
    own |diag T| / e_k move beyond 1/100 of the parity rule, the case is
    treated as ill-posed and only the exact invariants are comparable.  p = 0 is always well posed."""
    import oracle
    if p <= 0:
        return True
    # two perturbed samples, each required within 1/100 of the parity rule: a
    # sample only estimates the sensitivity
    for s in (12345, 54321):
        rng = np.random.default_rng(s)
        A2 = np.asfortranarray(A * (1.0 + 1e-15 * rng.standard_normal(A.shape)))
        r2 = oracle.randutv(A2, b, q, seed, k_stop=k_stop, build_ortho=False, p=p)
        par = check_parity(r2["T"], ref["T"], ref["a_fro"], rtol_diag=1e-12, rtol_ek=1e-10)
        if not (par["diag_ok"] and par["ek_ok"]):
            return False
    return True
