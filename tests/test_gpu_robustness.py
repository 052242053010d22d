"""Robustness of the C ABI beyond the parity configs (VERDICT r01 / ADVICE r01):

* in-place factorization on pinned host buffers (T aliases A) when an
  optimistic CholeskyQR decision fails and the call re-stages A;
* concurrent calls from several streams and host threads on the cached
  workspace (ordered on the device, DESIGN.md §6 "Streams");
* per-device library state (a second device when one is present);
* panels taller than the cluster Householder leaf holds (m > 65,536 rows):
  TSQR + Householder reconstruction, as a direct panel QR against the oracle's
  reflectors and inside a rank-deficient tall factorization against the oracle.
"""
import math
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from util import EPS, check_parity, diag_blocks_ok, invariants  # noqa: E402

pytestmark = pytest.mark.gpu


def to_dev(A, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A).T)).to(dev).t()


def to_host(X):
    return X.detach().cpu().numpy()


def low_rank(m, n, r, seed):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((m, r)) @ rng.standard_normal((r, n)))


def test_inplace_pinned_host_with_panel_fallback():
    """ADVICE r01 (driver.cu:852): T == A in pinned host memory, U = V = NULL.
    A has exact rank 150 < n, so the column panels after step 2 are rank
    deficient, CholeskyQR2's acceptance fails and the optimistic run is redone;
    the redo must start again from the untouched input."""
    m, n, b, q, seed = 700, 600, 64, 1, 5
    A = low_rank(m, n, 150, 9)
    _, Td, _, info = P.randutv(to_dev(A), b, q, seed, with_uv=False)
    assert info.qr_fallbacks > 0                         # the retry path is exercised
    Ah = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory()   # (n, m) row-major = A column-major
    rc = P.factor_raw(m, n, Ah.data_ptr(), m, b, q, seed, 0, None, Ah.data_ptr(), None)
    assert rc == 0
    Th = Ah.t().numpy()
    Td = to_host(Td)
    assert np.array_equal(Th == 0.0, Td == 0.0)
    assert np.abs(Th - Td).max() <= 1e-12 * np.linalg.norm(A)
    ref = oracle.randutv(A, b, q, seed, build_ortho=False)
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par


def test_concurrent_streams_and_threads():
    """Two user streams, then two host threads, each factoring on the cached
    workspace: every result equals the sequential one bitwise."""
    c = testmat.config("c2", scale=0.15)
    A = to_dev(c.A)
    _, T0, _, _ = P.randutv(A, c.b, c.q, c.seed, with_uv=False)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for s in (s1, s2, s1, s2):
        with torch.cuda.stream(s):
            _, T, _, _ = P.randutv(A, c.b, c.q, c.seed, with_uv=False, stream=s)
        outs.append(T)
    torch.cuda.synchronize()
    for T in outs:
        assert torch.equal(T, T0)
    res, errs = [None] * 4, []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                _, T, _, _ = P.randutv(A, c.b, c.q, c.seed, with_uv=False, stream=s)
                s.synchronize()
            res[i] = T
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    torch.cuda.synchronize()
    for T in res:
        assert torch.equal(T, T0)


def test_second_device_after_first():
    """Per-device workspace / attribute state: factor on cuda:0, then cuda:1,
    then cuda:0 again (skipped with a single GPU)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    c = testmat.config("c1", scale=0.5)
    ref = oracle.randutv(c.A, c.b, c.q, c.seed, build_ortho=False)
    for dev in ("cuda:0", "cuda:1", "cuda:0"):
        with torch.cuda.device(dev):
            _, T, _, _ = P.randutv(to_dev(c.A, dev), c.b, c.q, c.seed, with_uv=False)
            torch.cuda.synchronize()
        par = check_parity(to_host(T), ref["T"], ref["a_fro"])
        assert par["diag_ok"] and par["ek_ok"], (dev, par)


@pytest.mark.parametrize("m,b,degenerate", [(70000, 64, False), (100000, 128, False), (70000, 48, True)])
def test_panel_qr_taller_than_leaf(m, b, degenerate):
    """Householder mode on panels taller than the 16-CTA leaf (65,536 rows):
    TSQR of 8192-row chunks + Householder reconstruction.  Well-conditioned:
    the oracle's dlarfg reflectors, tau, R and T_w.  Degenerate (zero and
    repeated columns): a valid Householder QR (unit lower V, tau in [1, 2] or
    0, orthogonal Q, Q R = Y)."""
    rng = np.random.default_rng(m + b)
    Y = rng.standard_normal((m, b))
    if degenerate:
        Y[:, 5] = 0.0
        Y[:, 9] = Y[:, 8]
    V, R, tau, Tw, fb = P.panel_qr(to_dev(Y), mode=1, return_fallback=True)
    Vh, Th, Rh, th = to_host(V), to_host(Tw), to_host(R), to_host(tau)
    assert np.all(np.triu(Vh, 1) == 0) and np.all(np.diag(Vh) == 1) and np.all(np.tril(Rh, -1) == 0)
    Q1 = np.eye(m, b) - Vh @ (Th @ Vh[:b].T)
    assert np.linalg.norm(Q1.T @ Q1 - np.eye(b)) < 1e-13 * math.sqrt(m) * 10
    assert np.linalg.norm(Q1 @ Rh - Y) <= 1e-13 * np.linalg.norm(Y) * 10
    assert np.all(((th >= 1.0) & (th <= 2.0)) | (th == 0.0))
    if degenerate:
        return
    F, tau_o = oracle.geqr2(Y)
    Vo = oracle.unit_lower(F, b)
    To = oracle.larft(Vo, tau_o)
    Ro = np.triu(F[:b, :b])
    np.testing.assert_allclose(th, tau_o, rtol=0, atol=1e-12)
    np.testing.assert_allclose(Vh, Vo, rtol=0, atol=1e-10 * max(1, np.abs(Vo).max()))
    np.testing.assert_allclose(Rh, Ro, rtol=0, atol=1e-12 * np.abs(Ro).max())
    np.testing.assert_allclose(Th, To, rtol=0, atol=1e-10 * max(1, np.abs(To).max()))


@pytest.mark.parametrize("qr_mode", [0, 1])
def test_tall_rank_deficient_factorization_beyond_leaf(qr_mode):
    """m = 70,000 rows, exact rank 100 < n = 256: the column panels after step
    2 fail CholeskyQR2 (qr_mode 0) or are always Householder (qr_mode 1), and
    are taller than the leaf kernel -- the TSQR path -- against the oracle under
    R18, with the exact invariants."""
    m, n, b, q, seed = 70000, 256, 64, 1, 4
    A = low_rank(m, n, 100, 17)
    ref = oracle.randutv(A, b, q, seed, build_ortho=False)
    _, T, _, info = P.randutv(to_dev(A), b, q, seed, with_uv=False, qr_mode=qr_mode)
    torch.cuda.synchronize()
    Th = to_host(T)
    assert qr_mode == 1 or info.qr_fallbacks > 0
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert np.all(np.tril(Th, -1) == 0.0) and diag_blocks_ok(Th, b, n)
    assert abs(np.linalg.norm(Th) - np.linalg.norm(A)) <= 8 * m * EPS * np.linalg.norm(A)


def test_tall_factorization_with_uv_beyond_leaf():
    """The same TSQR panels with U and V formed (m = 66,000 > 65,536 rows,
    Householder only): A = U T V^T and orthogonality to 1e-13 n (n-scaled
    relative, the north star's invariants) on a thin 66,000 x 96 problem."""
    m, n, b, q, seed = 66000, 96, 32, 1, 2
    A = low_rank(m, n, 40, 23)
    U, T, V, info = P.randutv(to_dev(A), b, q, seed, with_uv=True, qr_mode=1)
    torch.cuda.synchronize()
    Uh, Th, Vh = to_host(U[:, :n]), to_host(T), to_host(V)
    # thin check (U is m x m): A = U(:, :n) T(:n, :) V^T since T(n:, :) = 0
    assert np.all(Th[n:, :] == 0.0)
    assert np.linalg.norm(A - Uh @ Th[:n] @ Vh.T) <= 1e-13 * n * np.linalg.norm(A)
    assert np.linalg.norm(Uh.T @ Uh - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Vh.T @ Vh - np.eye(n)) <= 1e-13 * n
    ref = oracle.randutv(A, b, q, seed, build_ortho=False)
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par


@pytest.mark.parametrize("uv,name,scale", [(False, "c2", 0.2), (True, "c1", 1.0), (False, "c4", 0.05)])
def test_graph_replay_bitwise(uv, name, scale):
    """A call repeated with the same arguments is captured into a CUDA graph on
    its second occurrence and replayed afterwards: every occurrence gives the
    same bits, and each counts the same number of kernel launches."""
    c = testmat.config(name, scale=scale)
    A = to_dev(c.A)
    m, n = c.A.shape
    T = P.empty_cm(m, n)
    U = P.empty_cm(m, m) if uv else None
    V = P.empty_cm(n, n) if uv else None
    outs, counts = [], []
    for _ in range(4):                                     # eager, capture, replay, replay
        l0 = P.launch_count()
        _, T, _, info = P.randutv(A, c.b, c.q, c.seed, with_uv=uv, out=(U, T, V))
        torch.cuda.synchronize()
        counts.append(P.launch_count() - l0)
        outs.append((T.clone(), U.clone() if uv else None, V.clone() if uv else None, info))
    for T_, U_, V_, info_ in outs[1:]:
        assert torch.equal(T_, outs[0][0])
        if uv:
            assert torch.equal(U_, outs[0][1]) and torch.equal(V_, outs[0][2])
        assert info_.k_done == outs[0][3].k_done and info_.steps == outs[0][3].steps
    assert len(set(counts)) == 1, counts
    # a different seed is a different graph: the result must change and match its own eager run
    _, T2, _, _ = P.randutv(A, c.b, c.q, c.seed + 1, with_uv=False)
    torch.cuda.synchronize()
    assert not torch.equal(T2, outs[0][0])
    ref = oracle.randutv(c.A, min(c.b, m, n), c.q, c.seed, build_ortho=False)
    par = check_parity(to_host(outs[-1][0]), ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par


@pytest.mark.parametrize("pin", [True, False])
def test_host_input_with_leading_dimension(pin):
    """Host A with lda > m (staged by the 2-D copy) against the contiguous host call
    (staged by one linear copy): the same bytes reach the device, so T is bitwise equal;
    pinned T (streamed copy-back, also of the tail chunks) and pageable T."""
    m, n, b, q, pad = 1100, 900, 64, 1, 7
    A = testmat.gaussian(m, n, 77)
    Ac = torch.from_numpy(np.ascontiguousarray(A.T))                # (n, m): column-major A, lda = m
    Ap = torch.full((n, m + pad), float("nan"), dtype=torch.float64)  # lda = m + pad, NaN in the padding
    Ap[:, :m] = Ac
    T1 = torch.empty(n, m, dtype=torch.float64)
    T2 = torch.empty(n, m, dtype=torch.float64)
    if pin:
        Ac, Ap, T1, T2 = Ac.pin_memory(), Ap.pin_memory(), T1.pin_memory(), T2.pin_memory()
    assert P.factor_raw(m, n, Ac.data_ptr(), m, b, q, 5, 0, None, T1.data_ptr(), None) == 0
    assert P.factor_raw(m, n, Ap.data_ptr(), m + pad, b, q, 5, 0, None, T2.data_ptr(), None) == 0
    assert torch.equal(T1, T2)
    assert bool(torch.isfinite(T1).all())
    assert diag_blocks_ok(T1.t().numpy()[:n, :n], b, n)


@pytest.mark.parametrize("m,n,b,q", [(3000, 3000, 64, 1), (2600, 2000, 128, 2)])
def test_pinned_host_copy_back_ordering(m, n, b, q):
    """Host-staged calls copy T's finished column blocks back while the loop
    runs; the copies must be ordered after the folds on the factorization's
    internal stream (a copy ordered on the caller's stream raced with them and
    returned undiagonalised blocks).  Every b x b diagonal block diagonal and
    equal to the device path's to rounding."""
    A = testmat.gaussian(m, n, m + n + b)
    Ah = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory()
    Th = torch.empty(n, m, dtype=torch.float64).pin_memory()
    for _ in range(2):
        rc = P.factor_raw(m, n, Ah.data_ptr(), m, b, q, 9, 0, None, Th.data_ptr(), None)
        assert rc == 0
        _, Td, _, _ = P.randutv(to_dev(A), b, q, 9, with_uv=False)
        torch.cuda.synchronize()
        Tp, Td = Th.t().numpy(), to_host(Td)
        k = min(m, n)
        assert diag_blocks_ok(Tp[:k, :k], b, k)
        assert np.array_equal(Tp == 0.0, Td == 0.0)
        assert np.abs(Tp - Td).max() <= 1e-12 * np.linalg.norm(A)
