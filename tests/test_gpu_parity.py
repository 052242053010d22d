"""GPU parity: every CUDA kernel and the whole factorization, through the C ABI,
against the oracle on the same seeded inputs (DESIGN.md §"Parity")."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from util import EPS, check_parity, diag_blocks_ok, ek_fro, invariants  # noqa: E402
from paper_1703_00998_b200 import dist as D_  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def to_dev(A: np.ndarray):
    """Column-major device copy of a host matrix."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A).T)).to(DEV).t()


def to_host(X):
    return X.detach().cpu().numpy()


# ----------------------------------------------------------------------------- Philox G
@pytest.mark.parametrize("rows,cols,seed,step", [(1, 1, 0, 0), (501, 50, 0, 3), (10000, 256, 3, 17),
                                                 (7, 5, 2**40 + 5, 1)])
def test_gaussian_matches_oracle(rows, cols, seed, step):
    g = to_host(P.gaussian(rows, cols, seed, step))
    r = oracle.gaussian_block(seed, step, rows, cols)
    ulp = np.spacing(np.abs(r))
    assert np.all(np.abs(g - r) <= 4 * ulp)            # transcendental libm vs CUDA: <= 4 ulp
    assert np.mean(g == r) > 0.5                        # most entries bitwise equal


# ----------------------------------------------------------------------------- DMMA GEMM
GEMM_CASES = [
    # (M, N, K, ta, tb)
    (1, 1, 1, False, False), (37, 29, 41, False, False), (130, 257, 33, True, False), (255, 129, 300, False, True),
    (128, 128, 16, True, True), (2000, 256, 3000, True, False), (32, 256, 10000, True, False),
    (3001, 513, 256, False, True), (64, 64, 0, False, False),
    # even leading dimensions, ragged M / N / K: the TMA-staged tiles (zero-filled edges)
    (1002, 250, 998, False, False), (1002, 250, 998, True, False), (1002, 250, 998, False, True),
    (1002, 250, 998, True, True), (2050, 1090, 300, False, True),
]


@pytest.mark.parametrize("M,N,K,ta,tb", GEMM_CASES)
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_dgemm_vs_oracle_matmul(M, N, K, ta, tb, beta):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((M, N))
    alpha = -1.25
    ref = alpha * (A.T if ta else A) @ (B.T if tb else B) + beta * C0
    C = to_dev(C0)
    P.dgemm(ta, tb, alpha, to_dev(A), to_dev(B), beta, C)
    got = to_host(C)
    bound = (K + 2) * EPS * (np.abs(A.T if ta else A) @ np.abs(B.T if tb else B) * abs(alpha) + abs(beta) * np.abs(C0))
    assert np.all(np.abs(got - ref) <= 2 * bound + 1e-300)


def test_dgemm_tma_path():
    """The TMA-staged tile variant (RANDUTV_GEMM_TMA=1, profiles/r02_tma_ab.md) on the same
    parity cases, in a fresh process (the switch is read once per process)."""
    import subprocess
    import sys
    import os
    env = dict(os.environ, RANDUTV_GEMM_TMA="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "test_dgemm_vs_oracle_matmul"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("env", [
    {"RANDUTV_GEMM_CLUSTER": "0"},                              # HBM partials + splitk_reduce
    {"RANDUTV_GEMM_CLUSTER": "1"},                              # cluster epilogue, partial-costed plans
    {"RANDUTV_GEMM_CLUSTER": "3"},                              # cluster epilogue on every <= 8-split grid
    {"RANDUTV_GEMM_CLUSTER": "3", "RANDUTV_GEMM_SPLITS": "3"},  # forced split counts through the cluster
    {"RANDUTV_GEMM_CLUSTER": "3", "RANDUTV_GEMM_SPLITS": "8"},
    {"RANDUTV_GEMM_CLUSTER": "3", "RANDUTV_GEMM_SPLITS": "8", "RANDUTV_GEMM_TMA": "1"},  # TMA tiles
    {"RANDUTV_GEMM_SPLITS": "12"},                              # > 8 splits: the partial workspace
])
def test_dgemm_split_k_paths(env):
    """The split-K variants (DSMEM cluster reduction, HBM partials) on the same
    parity cases, each in a fresh process (the switches are read once)."""
    import subprocess
    import sys
    import os
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "test_dgemm_vs_oracle_matmul or test_dgemm_misaligned_views"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_dgemm_misaligned_views():
    """Odd leading dimensions and odd offsets take the 8-byte load path."""
    rng = np.random.default_rng(1)
    big = to_dev(rng.standard_normal((301, 203)))
    A = big[1:150, 3:120]            # 149 x 117, ld 301, odd offset
    B = big[5:122, 7:40]             # 117 x 33
    C = torch.zeros(149, 33, dtype=torch.float64, device=DEV).t().contiguous().t()
    P.dgemm(False, False, 1.0, A, B, 0.0, C)
    ref = to_host(A) @ to_host(B)
    np.testing.assert_allclose(to_host(C), ref, rtol=0, atol=1e-12 * np.abs(ref).max())


# ----------------------------------------------------------------------------- Householder panel QR
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("m,b,decades", [(40, 8, 3), (500, 50, 3), (1000, 77, 3), (3000, 128, 3), (10000, 256, 3),
                                         (20000, 64, 3), (600, 512, 2), (5000, 200, 12)])
def test_panel_qr_vs_oracle(m, b, decades, mode):
    """mode 0 = CholeskyQR2 + Householder reconstruction (R20), mode 1 =
    column-by-column Householder; both must give the oracle's dlarfg reflectors.
    A 12-decade panel (kappa ~ 1e12) is beyond CholeskyQR2 and must take the
    Householder fallback in mode 0."""
    rng = np.random.default_rng(m + b)
    # graded columns mixed by a Haar rotation: kappa(Y) ~ 10^decades even after
    # column equilibration (column scaling alone leaves CholeskyQR accurate)
    H, _ = np.linalg.qr(rng.standard_normal((b, b)))
    Y = rng.standard_normal((m, b)) @ np.diag(10.0 ** -np.linspace(0, decades, b)) @ H
    V, R, tau, Tw, fb = P.panel_qr(to_dev(Y), mode=mode, return_fallback=True)
    assert fb == (mode == 0 and decades > 6)
    if decades > 6:
        # kappa ~ 1e12: the reflectors themselves are determined only to ~kappa eps;
        # check the factorization (structure, orthogonality, reconstruction)
        Vh, Th, Rh = to_host(V), to_host(Tw), to_host(R)
        assert np.all(np.triu(Vh, 1) == 0) and np.all(np.diag(Vh) == 1) and np.all(np.tril(Rh, -1) == 0)
        Q1 = np.eye(m, b) - Vh @ (Th @ Vh[:b].T)
        assert np.linalg.norm(Q1.T @ Q1 - np.eye(b)) < 1e-13 * math.sqrt(m) * 10
        assert np.linalg.norm(Q1 @ Rh - Y) <= 1e-13 * np.linalg.norm(Y) * 10
        assert np.all((to_host(tau) >= 1.0) & (to_host(tau) <= 2.0))
        return
    F, tau_o = oracle.geqr2(Y)
    Vo = oracle.unit_lower(F, b)
    To = oracle.larft(Vo, tau_o)
    Ro = np.triu(F[:b, :b])
    np.testing.assert_allclose(to_host(tau), tau_o, rtol=0, atol=1e-12)
    np.testing.assert_allclose(to_host(V), Vo, rtol=0, atol=1e-10 * max(1, np.abs(Vo).max()))
    np.testing.assert_allclose(to_host(R), Ro, rtol=0, atol=1e-12 * np.abs(Ro).max())
    np.testing.assert_allclose(to_host(Tw), To, rtol=0, atol=1e-10 * max(1, np.abs(To).max()))
    Vh, Th = to_host(V), to_host(Tw)
    assert np.all(np.triu(Vh, 1) == 0) and np.all(np.diag(Vh) == 1) and np.all(np.tril(to_host(R), -1) == 0)
    # orthogonality of the compact-WY product and reconstruction Y = Q [R; 0]
    Q1 = np.eye(m, b) - Vh @ (Th @ Vh[:b].T)
    assert np.linalg.norm(Q1.T @ Q1 - np.eye(b)) < 1e-13 * math.sqrt(m) * 10
    assert np.linalg.norm(Q1 @ to_host(R) - Y) <= 1e-13 * np.linalg.norm(Y) * 10


def test_panel_qr_degenerate_columns():
    """Zero and repeated columns: tau = 0 reflectors (H = I), still exact."""
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((300, 40))
    Y[:, 5] = 0.0
    Y[:, 9] = Y[:, 8]
    Y[:, 30:] = 0.0
    V, R, tau, Tw = P.panel_qr(to_dev(Y))
    F, tau_o = oracle.geqr2(Y)
    np.testing.assert_allclose(to_host(tau)[:5], tau_o[:5], atol=1e-13)
    assert np.all(to_host(tau)[30:] == 0.0)
    Vh, Th = to_host(V), to_host(Tw)
    Q1 = np.eye(300, 40) - Vh @ (Th @ Vh[:40].T)
    assert np.linalg.norm(Q1 @ to_host(R) - Y) <= 1e-12 * np.linalg.norm(Y)


# ----------------------------------------------------------------------------- batched Jacobi SVD
@pytest.mark.parametrize("k,batch", [(1, 2), (2, 3), (50, 4), (128, 3), (256, 2), (512, 1)])
def test_small_svd_batched_vs_lapack(k, batch):
    rng = np.random.default_rng(k)
    Rs = np.stack([np.triu(rng.standard_normal((k, k))) @ np.diag(10.0 ** -np.linspace(0, 5 * (i % 2), k))
                   for i in range(batch)])
    D, Us, Vs, sw = P.small_svd_batched(torch.from_numpy(Rs).to(DEV))
    D, Us, Vs = to_host(D), to_host(Us), to_host(Vs)
    for i in range(batch):
        s = oracle.small_svd(Rs[i])[1]
        np.testing.assert_allclose(D[i], s, rtol=0, atol=1e-13 * s[0] * max(1, k / 64))
        assert np.all(np.diff(D[i]) <= 0)
        assert np.linalg.norm(Us[i].T @ Us[i] - np.eye(k)) < 1e-12 * k
        assert np.linalg.norm(Vs[i].T @ Vs[i] - np.eye(k)) < 1e-12 * k
        assert np.linalg.norm(Us[i] @ np.diag(D[i]) @ Vs[i].T - Rs[i]) < 1e-13 * k * np.linalg.norm(Rs[i])
    assert to_host(sw).max() <= 40


def test_small_svd_closed_forms_and_zero():
    R = np.stack([np.array([[1.0, 1.0], [0.0, 1.0]]), np.zeros((2, 2)), np.array([[0.0, 1.0], [1.0, 0.0]])])
    D, Us, Vs, _ = P.small_svd_batched(torch.from_numpy(R).to(DEV))
    D, Us, Vs = to_host(D), to_host(Us), to_host(Vs)
    np.testing.assert_allclose(D[0], [(1 + 5 ** 0.5) / 2, (5 ** 0.5 - 1) / 2], rtol=1e-15)
    assert np.all(D[1] == 0)
    np.testing.assert_allclose(Vs[1].T @ Vs[1], np.eye(2), atol=1e-15)   # completed basis
    np.testing.assert_allclose(D[2], [1, 1], rtol=1e-15)
    for i in range(3):
        np.testing.assert_allclose(Us[i] @ np.diag(D[i]) @ Vs[i].T, R[i], atol=1e-15)


# ----------------------------------------------------------------------------- whole factorization
PARITY = [
    # name, scale, q override, with_uv
    ("c1", 1.0, None, True),      # BASELINE config 1 itself: 500 x 500, b=50, q=1
    ("c2", 0.2, 0, True),         # 600 x 600 exponential decay, b=128, q = 0/1/2
    ("c2", 0.2, 1, False),
    ("c2", 0.2, 2, True),
    ("c3", 0.1, None, False),     # 1000 x 1000 S-shape, b=125, q=2
    ("c4", 0.05, None, True),     # 1000 x 400 tall Gaussian, b=50, q=1 (tall final block)
]


@pytest.mark.parametrize("name,scale,q,uv,qr_mode", [p + (0,) for p in PARITY] + [
    ("c2", 0.2, 2, True, 1), ("c3", 0.1, None, False, 1), ("c4", 0.05, None, True, 1)])
def test_randutv_parity(name, scale, q, uv, qr_mode):
    """qr_mode 0: CholeskyQR2 + reconstruction panel QRs (default); 1: Householder."""
    c = testmat.config(name, scale=scale, q=q)
    A = c.A
    m, n = A.shape
    ref = oracle.randutv(A, c.b, c.q, c.seed, build_ortho=uv)
    U, T, V, info = P.randutv(to_dev(A), c.b, c.q, c.seed, with_uv=uv, qr_mode=qr_mode)
    torch.cuda.synchronize()
    Th = to_host(T)
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"], par
    assert par["ek_ok"], par
    assert info.k_done == n and info.steps == ref["steps"]
    assert np.all(np.tril(Th, -1) == 0.0)
    assert diag_blocks_ok(Th, c.b, n)
    inv = invariants(A, to_host(U) if uv else None, Th, to_host(V) if uv else None)
    assert inv["fro_rel"] <= n * EPS * 4
    if uv:
        assert inv["recon"] <= 1e-13 * n
        assert inv["orth_u"] <= 1e-13 * n and inv["orth_v"] <= 1e-13 * n


def test_randutv_ragged_and_b_geq_n():
    A = testmat.gaussian(333, 150, 11)
    for b in (32, 150, 400):
        ref = oracle.randutv(A, b, 1, 5)
        U, T, V, info = P.randutv(to_dev(A), b, 1, 5)
        par = check_parity(to_host(T), ref["T"], ref["a_fro"])
        assert par["diag_ok"] and par["ek_ok"], (b, par)
        inv = invariants(A, to_host(U), to_host(T), to_host(V))
        assert inv["recon"] < 1e-13 * 150 and inv["tril_max"] == 0


def test_randutv_early_stop_c5_like():
    """Config-5 shape at small scale: low rank + 1e-8 noise, k_stop and tol."""
    c = testmat.config("c5", scale=0.05)     # 1500 x 1500, rank 100, b=93, k_stop 102 -> k = 186
    ref = oracle.randutv(c.A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, build_ortho=False)
    U, T, V, info = P.randutv(to_dev(c.A), c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False)
    Th = to_host(T)
    assert info.k_done == ref["k"] and info.steps == ref["steps"]
    k = info.k_done
    assert np.all(Th[k:, :k] == 0)
    np.testing.assert_allclose(np.abs(np.diag(Th)[:k]), np.abs(np.diag(ref["T"])[:k]), rtol=1e-10,
                               atol=c.A.shape[0] * EPS * ref["a_fro"])
    assert abs(info.trailing_fro - ref["trailing_fro"]) <= 1e-8 * ref["trailing_fro"] + 1e3 * EPS * ref["a_fro"]


def test_identity_zero_and_nonfinite():
    n = 96
    U, T, V, _ = P.randutv(to_dev(np.eye(n)), 16, 1, 0)
    np.testing.assert_allclose(to_host(T), np.eye(n), atol=1e-13)
    U, T, V, _ = P.randutv(to_dev(np.zeros((n, n))), 16, 1, 0)
    assert np.all(to_host(T) == 0)
    assert np.linalg.norm(to_host(U).T @ to_host(U) - np.eye(n)) < 1e-12
    bad = np.ones((n, n)); bad[3, 4] = np.nan
    with pytest.raises(P.RandUTVError) as e:
        P.randutv(to_dev(bad), 16, 1, 0)
    assert e.value.code == 1


def test_host_buffers_match_device():
    """The C ABI on host buffers (staged inside the call) gives the same bits."""
    c = testmat.config("c1", scale=0.4)
    Uh, Th, Vh, _ = P.randutv(np.asfortranarray(c.A), c.b, c.q, c.seed)
    U, T, V, _ = P.randutv(to_dev(c.A), c.b, c.q, c.seed)
    assert np.array_equal(Th, to_host(T)) and np.array_equal(Uh, to_host(U))


def test_pinned_host_buffers_overlapped_copy_back():
    """T-only on PINNED host buffers: the folds of each SVD chunk are applied
    inside the loop and T's finished column blocks are copied back while the
    factorization runs (23 steps = several chunks, several copies).  The device
    path folds at the end, so the two agree to rounding (left and right
    products applied in a different order), with identical exact zeros."""
    A = testmat.gaussian(1500, 1500, 21)
    b, q, seed = 64, 1, 3
    m, n = A.shape
    Ah = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory()   # (n, m) row-major = A column-major
    Th = torch.empty(n, m, dtype=torch.float64).pin_memory()
    rc = P.factor_raw(m, n, Ah.data_ptr(), m, b, q, seed, 0, None, Th.data_ptr(), None)
    assert rc == 0
    _, T, _, _ = P.randutv(to_dev(A), b, q, seed, with_uv=False)
    Th, T = Th.t().numpy(), to_host(T)
    assert np.array_equal(Th == 0.0, T == 0.0)
    assert np.abs(Th - T).max() <= 1e-12 * np.linalg.norm(A)
    ref = oracle.randutv(A, b, q, seed, build_ortho=False)
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par


def test_deterministic():
    c = testmat.config("c2", scale=0.1)
    _, T1, _, _ = P.randutv(to_dev(c.A), c.b, c.q, c.seed, with_uv=False)
    _, T2, _, _ = P.randutv(to_dev(c.A), c.b, c.q, c.seed, with_uv=False)
    assert torch.equal(T1, T2)


# ----------------------------------------------------------------------------- over-sampling (NEXT row 1)
@pytest.mark.parametrize("name,scale,q,p,uv", [("c1", 1.0, None, 5, True), ("c2", 0.2, 1, 10, False),
                                                ("c2", 0.3, 2, 7, False), ("c4", 0.05, None, 3, True)])
def test_randutv_oversampling_parity(name, scale, q, p, uv):
    """Remark remark:positivep / Fig. fig:stepUTVoversampling on the GPU (QR of the
    extended Y, Jacobi SVD of its R factor, Z = Q Us(:, 1:b)) vs the oracle's
    LAPACK-SVD transcription; R23 caps p_i = min(p, n_i - b).  Parity needs the
    selection of the b dominant directions of Y' to be well posed
    (sigma_b(Y') / sigma_1(Y') >> eps, R23): spectra decaying by <= ~2 decades
    per block (c1, c2, c4; full-size c3 in test_gpu_fullsize)."""
    c = testmat.config(name, scale=scale, q=q)
    A = c.A
    m, n = A.shape
    ref = oracle.randutv(A, c.b, c.q, c.seed, build_ortho=uv, p=p)
    U, T, V, info = P.randutv(to_dev(A), c.b, c.q, c.seed, with_uv=uv, oversample=p)
    torch.cuda.synchronize()
    Th = to_host(T)
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert np.all(np.tril(Th, -1) == 0.0) and diag_blocks_ok(Th, c.b, n)
    if uv:
        inv = invariants(A, to_host(U), Th, to_host(V))
        assert inv["recon"] <= 1e-13 * n and inv["orth_u"] <= 1e-13 * n and inv["orth_v"] <= 1e-13 * n


def test_oversampling_argument_checks():
    A = to_dev(testmat.gaussian(64, 64, 1))
    with pytest.raises(P.RandUTVError):
        P.randutv(A, 16, 1, 0, oversample=-1)
    with pytest.raises(P.RandUTVError):
        P.randutv(A, 256, 1, 0, oversample=300)     # b + p > RANDUTV_MAX_B


# ----------------------------------------------------------------------------- fat inputs (NEXT row 2)
@pytest.mark.parametrize("m,n,b,q,uv", [(300, 500, 50, 1, True), (400, 1000, 64, 1, False), (130, 400, 32, 2, True),
                                        (100, 333, 128, 1, True), (256, 300, 50, 1, False)])
def test_randutv_fat_parity(m, n, b, q, uv):
    """m < n (Remark "The case m < n"): the randomized steps as for
    m >= n, the final fat block by a QR of its rows (transpose + panel QR), its
    triangular factor's SVD, and V's last factor = the row reflectors."""
    A = testmat.gaussian(m, n, m + n)
    ref = oracle.randutv(A, b, q, 7, build_ortho=uv)
    U, T, V, info = P.randutv(to_dev(A), b, q, 7, with_uv=uv)
    torch.cuda.synchronize()
    Th = to_host(T)
    par = check_parity(Th, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert info.k_done == m and info.final_block and np.all(np.tril(Th, -1) == 0.0)
    assert np.all(Th[:, m:][np.arange(m) >= (m // b) * b if m % b else np.zeros(m, bool)] == 0)
    if uv:
        inv = invariants(A, to_host(U), Th, to_host(V))
        assert inv["recon"] <= 1e-13 * n and inv["orth_u"] <= 1e-13 * n and inv["orth_v"] <= 1e-13 * n


# ----------------------------------------------------------------------------- randomized SVD (NEXT row 3)
@pytest.mark.parametrize("m,n,b,q,p,decay", [(500, 400, 50, 1, 0, 0.99), (1000, 800, 64, 2, 10, 0.97),
                                             (3000, 2000, 128, 1, 5, 0.995), (600, 700, 96, 0, 0, 0.98)])
def test_rsvd_vs_oracle(m, n, b, q, p, decay):
    """randutv_rsvd (Remark remark:RSVD) vs the oracle on the same Philox G:
    D within the parity rule, the approximation error ||A - U D V^T||_F within
    1e-8 relative, U and V orthonormal."""
    rng = np.random.default_rng(m + n)
    k = min(m, n)
    s = decay ** np.arange(k)
    A = (np.linalg.qr(rng.standard_normal((m, k)))[0] * s) @ np.linalg.qr(rng.standard_normal((n, k)))[0].T
    Uo, Do, Vo, _ = oracle.rsvd(A, b, q, seed=11, p=p)
    U, D, V = P.rsvd(to_dev(A), b, q, 11, oversample=p)
    torch.cuda.synchronize()
    U, D, V = to_host(U), to_host(D), to_host(V)
    a = np.linalg.norm(A)
    floor = max(m, n) * EPS * a
    assert np.all(np.abs(D - Do) <= 1e-10 * Do + floor)
    e_gpu = np.linalg.norm(A - (U * D) @ V.T)
    e_orc = np.linalg.norm(A - (Uo * Do) @ Vo.T)
    assert abs(e_gpu - e_orc) <= 1e-8 * e_orc + floor
    assert np.linalg.norm(U.T @ U - np.eye(b)) < 1e-13 * m and np.linalg.norm(V.T @ V - np.eye(b)) < 1e-13 * n
    assert np.all(np.diff(D) <= 0)


def test_poisoned_workspace_initcheck():
    """compute-sanitizer is closed on the GPU pool; instead every workspace is
    filled with NaN bit patterns before use (RANDUTV_POISON_WORKSPACE), so a
    kernel reading workspace memory it never wrote would put NaN into the
    results.  Outputs must be finite and equal to the normal run."""
    import os
    c = testmat.config("c1")
    A2 = testmat.gaussian(700, 520, 9)
    runs = []
    for poison in (False, True):
        if poison:
            os.environ["RANDUTV_POISON_WORKSPACE"] = "1"
        try:
            out = []
            U, T, V, _ = P.randutv(to_dev(c.A), c.b, c.q, c.seed)
            out += [U, T, V]
            _, T2, _, _ = P.randutv(to_dev(A2), 64, 2, 4, with_uv=False, oversample=6)
            _, T3, _, _ = P.randutv(to_dev(A2), 64, 1, 4, with_uv=False, qr_mode=1)
            out += [T2, T3]
            Uk, D, Vk = P.rsvd(to_dev(A2), 48, 1, 5)
            out += [Uk, D, Vk]
            comm = D_.loopback(3)
            sh = [D_.shard(to_dev(A2), 64, r, 3) for r in range(3)]
            Us, Ts, Vs, _ = D_.factor(comm, sh, 700, 520, 64, 1, 2, with_uv=True)
            comm.close()
            out += [D_.assemble(Us, 700, 64), D_.assemble(Ts, 520, 64), D_.assemble(Vs, 520, 64)]
            comm = D_.loopback(2)
            sh = [D_.shard(to_dev(A2), 64, r, 2) for r in range(2)]
            Ts, _ = D_.factor(comm, sh, 700, 520, 64, 2, 3, oversample=6)
            comm.close()
            out += [D_.assemble(Ts, 520, 64)]
            A3 = to_dev(testmat.gaussian(300, 640, 4))   # fat: the final block spans the ranks
            comm = D_.loopback(3)
            sh = [D_.shard(A3, 64, r, 3) for r in range(3)]
            Us, Ts, Vs, _ = D_.factor(comm, sh, 300, 640, 64, 1, 5, with_uv=True)
            comm.close()
            out += [D_.assemble(Us, 300, 64), D_.assemble(Ts, 640, 64), D_.assemble(Vs, 640, 64)]
            torch.cuda.synchronize()
            runs.append([to_host(x) for x in out])
        finally:
            os.environ.pop("RANDUTV_POISON_WORKSPACE", None)
    for a, p in zip(*runs):
        assert np.all(np.isfinite(p))
        assert np.array_equal(a, p)


@pytest.mark.parametrize("m,n", [(149, 19), (85, 38), (24, 128), (34, 300), (400, 256)])
def test_final_block_r_factor_accuracy(m, n):
    """b >= min(m, n): the whole matrix is the final block, whose Householder R
    factor is kept in T.  With kappa ~ 3e7 (inside CholeskyQR2's range, where
    its R is no longer backward stable) the panel QR must fall back to
    Householder (QrWork::orth_tol = kRFactorOrthTol): |diag T| equal to the
    singular values to O(k eps ||A||) (was ~1e-11 off before the tolerance)."""
    rng = np.random.default_rng(m * 1000 + n)
    k = min(m, n)
    U, _ = np.linalg.qr(rng.standard_normal((m, k)))
    V, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s = np.logspace(0, -7.5, k)
    A = np.asfortranarray(U @ np.diag(s) @ V.T)
    _, T, _, info = P.randutv(to_dev(A), 512, 1, 3, with_uv=False)
    torch.cuda.synchronize()
    d = np.sort(np.abs(np.diag(to_host(T))[:k]))[::-1]
    sv = np.linalg.svd(A, compute_uv=False)
    assert np.abs(d - sv).max() <= 10 * k * EPS * sv[0], np.abs(d - sv).max()
