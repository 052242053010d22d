"""Randomised shapes through the whole GPU path against the oracle (DESIGN.md
R18 parity rule) and the exact invariants: tall, square and fat m x n, b from 1
to beyond n, q in 0..3, both QR modes, over-sampling, early stop, graded and
rank-deficient spectra.  Seeds are fixed (reproducible)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
from util import EPS, check_parity, selection_well_posed  # noqa: E402

pytestmark = pytest.mark.gpu


def to_dev(A):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A).T)).cuda().t()


def make(rng, m, n, kind):
    A = rng.standard_normal((m, n))
    k = min(m, n)
    if kind == "graded":
        U, _ = np.linalg.qr(rng.standard_normal((m, k)))
        V, _ = np.linalg.qr(rng.standard_normal((n, k)))
        A = U @ np.diag(np.logspace(0, -rng.uniform(2, 10), k)) @ V.T
    elif kind == "lowrank":
        r = max(1, k // 3)
        A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) + 1e-9 * rng.standard_normal((m, n))
    return np.asfortranarray(A)


CASES = []
_rng = np.random.default_rng(20261020)
for _ in range(60):
    m = int(_rng.integers(3, 420))
    n = int(_rng.integers(3, 420))
    b = int(_rng.choice([1, 2, 7, 16, 31, 48, 64, 100, 500]))
    q = int(_rng.integers(0, 4))
    kind = str(_rng.choice(["gauss", "graded", "lowrank"]))
    qr_mode = int(_rng.integers(0, 2))
    p = int(_rng.choice([0, 0, 0, 3]))
    k_stop = int(_rng.choice([0, 0, 0, b * 2]))
    seed = int(_rng.integers(0, 2**31))
    CASES.append((m, n, b, q, kind, qr_mode, p, k_stop, seed))


@pytest.mark.parametrize("m,n,b,q,kind,qr_mode,p,k_stop,seed", CASES)
def test_fuzz_vs_oracle(m, n, b, q, kind, qr_mode, p, k_stop, seed):
    rng = np.random.default_rng(seed)
    A = make(rng, m, n, kind)
    bb = min(b, m, n)
    if p > 0 and m < n:
        p = 0  # over-sampling with fat inputs is not supported (R8)
    if p > 0:
        p = min(p, max(0, min(m, n) - bb))
    ref = oracle.randutv(A, bb, q, seed, k_stop=k_stop, build_ortho=True, p=p)
    U, T, V, info = P.randutv(to_dev(A), b, q, seed, k_stop=k_stop, qr_mode=qr_mode, oversample=p)
    torch.cuda.synchronize()
    U, T, V = U.cpu().numpy(), T.cpu().numpy(), V.cpu().numpy()
    a = np.linalg.norm(A)
    assert np.all(np.isfinite(T)) and np.all(np.isfinite(U)) and np.all(np.isfinite(V))
    assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * max(m, n) * max(a, 1e-300)
    assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * max(m, n)
    assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * max(m, n)
    assert info.k_done == ref["k"]
    k = info.k_done
    assert np.all(np.tril(T[:, :k], -1) == 0.0)
    if p > 0 and not selection_well_posed(A, bb, q, seed, p, ref, k_stop=k_stop):
        return  # over-sampled selection ill-posed (R23): the invariants above are what is unique
    if kind != "lowrank":  # parity of |diag T|, e_k (rank-deficient tails are at the noise floor)
        par = check_parity(T, ref["T"], ref["a_fro"])
        assert par["diag_ok"] and par["ek_ok"], par
    else:
        d, dr = np.abs(np.diag(T)), np.abs(np.diag(ref["T"]))
        assert np.all(np.abs(d - dr) <= 1e-10 * dr + 1e-8 * a), np.max(np.abs(d - dr))
