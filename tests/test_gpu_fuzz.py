"""Randomised shapes through the whole GPU path against the oracle (DESIGN.md
R18 parity rule on every |t_jj| and e_k, for every input kind) and the exact
invariants: tall, square and fat m x n, b from 1 to beyond n, q in 0..3, both
QR modes, over-sampling (on graded spectra), early stop, Gaussian, graded and
rank-deficient inputs.  Cases: tests/fuzz_cases.py (fixed seeds)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
from fuzz_cases import CASES, effective, make  # noqa: E402
from util import EPS, check_parity, selection_well_posed  # noqa: E402

pytestmark = pytest.mark.gpu


def to_dev(A):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A).T)).cuda().t()


@pytest.mark.parametrize("m,n,b,q,kind,qr_mode,p,k_stop,seed", CASES)
def test_fuzz_vs_oracle(m, n, b, q, kind, qr_mode, p, k_stop, seed):
    rng = np.random.default_rng(seed)
    A = make(rng, m, n, kind)
    bb, p = effective(m, n, b, p)
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
        # over-sampled selection ill-posed (R23): the invariants above are what is
        # unique (at most 1/4 of these cases, tests/test_fuzz_design.py)
        return
    # every kind, rank-deficient included: R18 on every |t_jj| and every e_k
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
