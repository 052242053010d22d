"""Full BASELINE.json sizes, in the configuration bench.py times (T-only,
randutv_factor_ex on device buffers), checked against the oracle on outputs it
can compute at that size and on size-independent properties:

* c2 (3000^2, q = 0, 1, 2): the whole factorization against the oracle (R18).
* c3 (10000^2, q = 2) and c4 (20000 x 8000, q = 1): the first randomized step
  against the oracle run with k_stop = b on the same bytes -- T(1:b, 1:b) is
  final after step 1 and e_b = ||T(b+1:m, :)||_F is invariant under every
  later (orthogonal, row- or column-local) step; plus exact triangularity,
  ||T||_F = ||A||_F, diagonal blocks, and for c3 the determinant identity
  sum log|t_jj| = sum log sigma_j against the known spectrum.
* c5 (30000^2, b = 512, k_stop 2048, tol 1e-6): stops at k = 2048 with the
  trailing norm at the noise level, T(k:, :k) = 0.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from util import EPS, check_parity, diag_blocks_ok  # noqa: E402

pytestmark = pytest.mark.gpu


def device_case(name, q=None):
    At, c = testmat.device_config(name)
    if q is not None:
        c.q = q
    return At.t(), c


def factor_T(A, c):
    m, n = A.shape
    T = P.empty_cm(m, n)
    _, T, _, info = P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None))
    torch.cuda.synchronize()
    return T, info


def first_step_checks(A, T, c):
    """Oracle with k_stop = b on the same bytes vs the GPU's full factorization."""
    Ah = np.asfortranarray(A.cpu().numpy())
    ref = oracle.randutv(Ah, c.b, c.q, c.seed, k_stop=c.b, build_ortho=False)
    b = c.b
    floor = max(Ah.shape) * EPS * ref["a_fro"]
    d_gpu = torch.diagonal(T[:b, :b]).abs().cpu().numpy()
    d_ref = np.abs(np.diag(ref["T"])[:b])
    assert np.all(np.abs(d_gpu - d_ref) <= 1e-10 * d_ref + floor), np.max(np.abs(d_gpu - d_ref) / d_ref)
    e_gpu = torch.linalg.norm(T[b:, :]).item()
    e_ref = float(np.linalg.norm(ref["T"][b:, :]))
    assert abs(e_gpu - e_ref) <= 1e-8 * e_ref + floor, (e_gpu, e_ref)
    return ref["a_fro"]


def structure_checks(A, T, c, k):
    m, n = A.shape
    assert torch.count_nonzero(torch.tril(T[:, :k], -1)).item() == 0          # exact zeros (R12)
    a_fro = torch.linalg.norm(A).item()
    assert abs(torch.linalg.norm(T).item() - a_fro) <= 8 * max(m, n) * EPS * a_fro
    Tk = T[:k, :k].cpu().numpy()
    assert diag_blocks_ok(Tk, c.b, k)


@pytest.mark.parametrize("q", [0, 1, 2])
def test_c2_full_vs_oracle(q):
    A, c = device_case("c2", q=q)
    T, info = factor_T(A, c)
    Ah = np.asfortranarray(A.cpu().numpy())
    ref = oracle.randutv(Ah, c.b, c.q, c.seed, build_ortho=False)
    par = check_parity(T.cpu().numpy(), ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert info.steps == ref["steps"] and info.k_done == A.shape[1]


def test_c3_full():
    A, c = device_case("c3")
    T, info = factor_T(A, c)
    n = A.shape[1]
    assert info.k_done == n and info.steps == 39 and info.final_block
    first_step_checks(A, T, c)
    structure_checks(A, T, c, n)
    # |det T| = |det A| = prod sigma_j (square A, orthogonal U, V)
    logd = torch.log(torch.diagonal(T).abs()).sum().item()
    logs = float(np.sum(np.log(c.sigma)))
    assert abs(logd - logs) <= 1e-6 * abs(logs) + 1e-3, (logd, logs)
    # the randomized blocks reveal the spectrum: t_jj within the band of
    # SURVEY App. A.4b (one-sided: the flat region is never over-estimated)
    d = torch.diagonal(T).abs().cpu().numpy()
    assert np.all(d[:2000] <= c.sigma[:2000] * (1 + 1e-9)) and np.all(d[:2000] >= 0.9 * c.sigma[:2000])
    assert np.all(d[3000:] >= 0.9 * c.sigma[3000:]) and np.all(d[3000:] <= 1.3 * c.sigma[3000:])


def test_c3_full_oversampled_first_step():
    """Over-sampling p = 10 at the c3 size: the first block against the oracle
    run with k_stop = b on the same bytes (R23: 2 decades per block keep the
    selection of Y's dominant directions well posed)."""
    A, c = device_case("c3")
    m, n = A.shape
    T = P.empty_cm(m, n)
    _, T, _, info = P.randutv(A, c.b, c.q, c.seed, k_stop=c.b, with_uv=False, out=(None, T, None), oversample=10)
    torch.cuda.synchronize()
    Ah = np.asfortranarray(A.cpu().numpy())
    ref = oracle.randutv(Ah, c.b, c.q, c.seed, k_stop=c.b, build_ortho=False, p=10)
    b = c.b
    floor = n * EPS * ref["a_fro"]
    d_gpu = torch.diagonal(T[:b, :b]).abs().cpu().numpy()
    d_ref = np.abs(np.diag(ref["T"])[:b])
    assert np.all(np.abs(d_gpu - d_ref) <= 1e-10 * d_ref + floor), np.max(np.abs(d_gpu - d_ref) / d_ref)
    assert abs(info.trailing_fro - ref["trailing_fro"]) <= 1e-8 * ref["trailing_fro"] + floor


def test_c4_full_tall():
    A, c = device_case("c4")
    T, info = factor_T(A, c)
    m, n = A.shape
    assert info.k_done == n and info.final_block and info.steps == 31
    first_step_checks(A, T, c)
    structure_checks(A, T, c, n)
    assert torch.count_nonzero(T[n:, :]).item() == 0


def test_c5_full_early_stop():
    A, c = device_case("c5")
    T, info = factor_T(A, c)
    k = info.k_done
    assert k == 2048 and info.steps == 4
    assert torch.count_nonzero(T[k:, :k]).item() == 0
    assert torch.count_nonzero(torch.tril(T[:k, :k], -1)).item() == 0
    assert diag_blocks_ok(T[:k, :k].cpu().numpy(), c.b, k)
    # rank 2000 < k: the trailing block is the 1e-8 noise (Frobenius ~ 1e-8 * 28000)
    noise = 1e-8 * (A.shape[0] - k)
    tr = torch.linalg.norm(T[k:, k:]).item()
    assert 0.5 * noise <= info.trailing_fro <= 2.0 * noise, (info.trailing_fro, noise)
    assert abs(tr - info.trailing_fro) <= 1e-6 * tr
    a_fro = torch.linalg.norm(A).item()
    assert info.trailing_fro <= c.tol * a_fro
