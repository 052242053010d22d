"""GPU parity of the multi-GPU algorithm (randutv_factor_dist) through the C
ABI, on ONE GPU with the loopback communicator: P virtual ranks, each with its
own block-cyclic shard, collectives as fixed-order device sums/copies between
bulk-synchronous phases.  The assembled T must satisfy the same parity rule
against the oracle as the single-GPU path (R18) and agree with the
single-GPU factorization to rounding."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from paper_1703_00998_b200 import dist as D  # noqa: E402
from util import EPS, check_parity, diag_blocks_ok, selection_well_posed  # noqa: E402

pytestmark = pytest.mark.gpu


def to_dev(A):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A).T)).cuda().t()


def run_dist(A, nranks, b, q, seed, **kw):
    m, n = A.shape
    comm = D.loopback(nranks)
    Ad = to_dev(A)
    shards = [D.shard(Ad, b, r, nranks) for r in range(nranks)]
    Ts, info = D.factor(comm, shards, m, n, b, q, seed, **kw)
    torch.cuda.synchronize()
    comm.close()
    return D.assemble(Ts, n, min(b, n)).cpu().numpy(), info


@pytest.mark.parametrize("name,scale,q,nranks", [
    ("c1", 1.0, None, 2), ("c1", 1.0, None, 3), ("c2", 0.2, 2, 4), ("c3", 0.1, None, 2),
    ("c3", 0.1, None, 8), ("c4", 0.05, None, 3)])
def test_dist_loopback_parity(name, scale, q, nranks):
    c = testmat.config(name, scale=scale, q=q)
    A = c.A
    m, n = A.shape
    ref = oracle.randutv(A, c.b, c.q, c.seed, build_ortho=False)
    T, info = run_dist(A, nranks, c.b, c.q, c.seed)
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert info.k_done == n and info.steps == ref["steps"]
    assert np.all(np.tril(T, -1) == 0.0)
    assert diag_blocks_ok(T, c.b, n)
    assert abs(np.linalg.norm(T) - np.linalg.norm(A)) <= 4 * n * EPS * np.linalg.norm(A)
    # the single-GPU path on the same input: equal to rounding
    _, T1, _, _ = P.randutv(to_dev(A), c.b, c.q, c.seed, with_uv=False)
    T1 = T1.cpu().numpy()
    d1, dd = np.abs(np.diag(T1)), np.abs(np.diag(T))
    assert np.all(np.abs(d1 - dd) <= 1e-10 * d1 + n * EPS * ref["a_fro"])


def test_dist_one_rank_equals_single_gpu_bits():
    """P = 1: the same kernels in the same order as randutv_factor_ex, except
    that the Grams go through the packed allreduce buffer -- equal to rounding."""
    c = testmat.config("c1", scale=0.4)
    T, info = run_dist(c.A, 1, c.b, c.q, c.seed)
    _, T1, _, _ = P.randutv(to_dev(c.A), c.b, c.q, c.seed, with_uv=False)
    np.testing.assert_allclose(np.abs(np.diag(T)), np.abs(np.diag(T1.cpu().numpy())), rtol=1e-12, atol=1e-13)


def test_dist_more_ranks_than_blocks_and_ragged():
    A = testmat.gaussian(333, 150, 11)
    for nranks, b in ((4, 64), (5, 32), (3, 150)):
        ref = oracle.randutv(A, b, 1, 5, build_ortho=False)
        T, info = run_dist(A, nranks, b, 1, 5)
        par = check_parity(T, ref["T"], ref["a_fro"])
        assert par["diag_ok"] and par["ek_ok"], (nranks, b, par)


def test_dist_early_stop_c5_like():
    c = testmat.config("c5", scale=0.05)
    ref = oracle.randutv(c.A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, build_ortho=False)
    T, info = run_dist(c.A, 3, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol)
    k = info.k_done
    assert k == ref["k"] and info.steps == ref["steps"]
    assert np.all(T[k:, :k] == 0)
    np.testing.assert_allclose(np.abs(np.diag(T)[:k]), np.abs(np.diag(ref["T"])[:k]), rtol=1e-10,
                               atol=c.A.shape[0] * EPS * ref["a_fro"])
    assert abs(info.trailing_fro - ref["trailing_fro"]) <= 1e-8 * ref["trailing_fro"] + 1e3 * EPS * ref["a_fro"]


def test_dist_householder_fallback_and_zero():
    """qr_mode 1 forces the allgather + redundant Householder path; a zero
    matrix triggers the CholeskyQR breakdown fallback in qr_mode 0."""
    c = testmat.config("c2", scale=0.1)
    ref = oracle.randutv(c.A, c.b, c.q, c.seed, build_ortho=False)
    T, info = run_dist(c.A, 3, c.b, c.q, c.seed, qr_mode=1)
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    Z, info = run_dist(np.zeros((96, 96)), 2, 16, 1, 0)
    assert np.all(Z == 0) and info.qr_fallbacks > 0


def test_dist_nccl_one_rank():
    """The NCCL communicator (unique id exchanged through torch.distributed,
    symbols from the process's libnccl) on a 1-rank group."""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29600 + os.getpid() % 500))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = D.nccl_from_torch()
        assert comm.world == 1 and comm.ranks == [0]
        c = testmat.config("c1", scale=0.4)
        ref = oracle.randutv(c.A, c.b, c.q, c.seed, build_ortho=False)
        Ts, info = D.factor(comm, [to_dev(c.A)], *c.A.shape, c.b, c.q, c.seed)
        torch.cuda.synchronize()
        par = check_parity(Ts[0].cpu().numpy(), ref["T"], ref["a_fro"])
        assert par["diag_ok"] and par["ek_ok"], par
        comm.close()
    finally:
        dist.destroy_process_group()


def run_dist_uv(A, nranks, b, q, seed, **kw):
    m, n = A.shape
    comm = D.loopback(nranks)
    Ad = to_dev(A)
    shards = [D.shard(Ad, b, r, nranks) for r in range(nranks)]
    Us, Ts, Vs, info = D.factor(comm, shards, m, n, b, q, seed, with_uv=True, **kw)
    torch.cuda.synchronize()
    comm.close()
    bb = min(b, n)
    U = D.assemble(Us, m, bb).cpu().numpy()
    T = D.assemble(Ts, n, bb).cpu().numpy()
    V = D.assemble(Vs, n, bb).cpu().numpy()
    return U, T, V, info


@pytest.mark.parametrize("m,n,b,q,nranks,kw", [
    (500, 500, 50, 1, 3, {}),                      # c1 shape
    (1000, 400, 64, 1, 2, {}),                     # tall: final tall block (QR + SVD)
    (333, 150, 64, 2, 4, {}),                      # ragged, a rank without V columns
    (600, 600, 64, 1, 3, {"k_stop": 192}),         # early stop: dense trailing block
    (384, 384, 128, 0, 2, {"qr_mode": 1}),         # Householder panels
])
def test_dist_uv_factorization(m, n, b, q, nranks, kw):
    """U and V formed on the shards (backward accumulation):
    A = U T V^T and orthogonality to the north star's 1e-13 n bound; T as in the
    T-only run against the oracle."""
    A = testmat.gaussian(m, n, m + n + nranks)
    U, T, V, info = run_dist_uv(A, nranks, b, q, 7, **kw)
    a = np.linalg.norm(A)
    assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * n * a
    assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * n
    assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * n
    ref = oracle.randutv(A, b, q, 7, build_ortho=False, **{k: v for k, v in kw.items() if k == "k_stop"})
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    # the T-only distributed run gives the same T to rounding
    T0, _ = run_dist(A, nranks, b, q, 7, **kw)
    np.testing.assert_allclose(T, T0, rtol=0, atol=1e-12 * a)


_drng = np.random.default_rng(7)
DIST_FUZZ = []
for _ in range(12):
    n = int(_drng.integers(8, 300))
    m = n + int(_drng.integers(0, 200))
    DIST_FUZZ.append((m, n, int(_drng.choice([4, 16, 33, 64])), int(_drng.integers(0, 3)), int(_drng.integers(1, 6)),
                      bool(_drng.integers(0, 2)), int(_drng.integers(0, 2**31))))


@pytest.mark.parametrize("m,n,b,q,nranks,uv,seed", DIST_FUZZ)
def test_dist_fuzz(m, n, b, q, nranks, uv, seed):
    """Random shapes, block widths and rank counts through the loopback
    communicator: T against the oracle's parity rule; with U, V the exact
    invariants."""
    A = testmat.gaussian(m, n, seed % 1000)
    ref = oracle.randutv(A, min(b, n), q, seed, build_ortho=False)
    if uv:
        U, T, V, info = run_dist_uv(A, nranks, b, q, seed)
        a = np.linalg.norm(A)
        assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * m * a
        assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * m
        assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * m
    else:
        T, info = run_dist(A, nranks, b, q, seed)
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert np.all(np.tril(T, -1) == 0.0)


@pytest.mark.parametrize("name,scale,q,p,nranks,uv", [("c1", 1.0, None, 5, 3, True), ("c2", 0.2, 1, 10, 2, False),
                                                      ("c2", 0.3, 2, 7, 4, False), ("c4", 0.05, None, 3, 3, True)])
def test_dist_oversampling_parity(name, scale, q, p, nranks, uv):
    """Over-sampling (R23) through the multi-GPU algorithm: the b + p_i column
    sketch is row-distributed; Z = Q U_R(:, 1:b) from the allgathered sketch.
    Same parity rule against the oracle's LAPACK-SVD transcription as the
    single-GPU test (test_randutv_oversampling_parity), and the single-GPU
    over-sampled run to rounding."""
    c = testmat.config(name, scale=scale, q=q)
    A = c.A
    m, n = A.shape
    ref = oracle.randutv(A, c.b, c.q, c.seed, build_ortho=False, p=p)
    if uv:
        U, T, V, info = run_dist_uv(A, nranks, c.b, c.q, c.seed, oversample=p)
        a = np.linalg.norm(A)
        assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * n * a
        assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * n
        assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * n
    else:
        T, info = run_dist(A, nranks, c.b, c.q, c.seed, oversample=p)
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert np.all(np.tril(T, -1) == 0.0) and diag_blocks_ok(T, c.b, n)
    _, T1, _, _ = P.randutv(to_dev(A), c.b, c.q, c.seed, with_uv=False, oversample=p)
    d1, dd = np.abs(np.diag(T1.cpu().numpy())), np.abs(np.diag(T))
    assert np.all(np.abs(d1 - dd) <= 1e-10 * d1 + n * EPS * ref["a_fro"])


def test_dist_oversampling_householder_reortho():
    """qr_mode 1: the re-orthonormalizations of the b + p_i column sketch take
    the allgather + redundant Householder path (width b + p_i), QR(Y) too."""
    c = testmat.config("c2", scale=0.2, q=2)
    ref = oracle.randutv(c.A, c.b, c.q, c.seed, build_ortho=False, p=9)
    T, info = run_dist(c.A, 3, c.b, c.q, c.seed, oversample=9, qr_mode=1)
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert info.qr_fallbacks > 0


def test_dist_oversampling_argument_checks():
    A = testmat.gaussian(64, 64, 1)
    with pytest.raises(Exception):
        run_dist(A, 2, 256, 1, 0, oversample=300)   # b + p > RANDUTV_MAX_B
    with pytest.raises(Exception):
        run_dist(A, 2, 16, 1, 0, oversample=-1)


_orng = np.random.default_rng(11)
DIST_OVS_FUZZ = []
for _ in range(16):
    n = int(_orng.integers(40, 900))
    m = n + int(_orng.integers(0, 300))
    DIST_OVS_FUZZ.append((m, n, int(_orng.choice([8, 15, 16, 33, 64, 100])), int(_orng.integers(0, 3)),
                          int(_orng.integers(1, 9)), int(_orng.integers(1, 13)), bool(_orng.integers(0, 2)),
                          int(_orng.integers(0, 2**31))))


@pytest.mark.parametrize("m,n,b,q,nranks,p,uv,seed", DIST_OVS_FUZZ)
def test_dist_oversampling_fuzz(m, n, b, q, nranks, p, uv, seed):
    """Random shapes / ranks / over-sampling p on Gaussian inputs: the exact
    invariants always; T against the oracle's parity rule where the
    b-of-(b + p_i) selection is well posed (selection_well_posed: flat
    trailing spectra can leave sigma_b(Y') ~ sigma_{b+1}(Y'), R23)."""
    A = testmat.gaussian(m, n, seed % 1000)
    ref = oracle.randutv(A, min(b, n), q, seed, build_ortho=False, p=p)
    if uv:
        U, T, V, info = run_dist_uv(A, nranks, b, q, seed, oversample=p)
        a = np.linalg.norm(A)
        assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * m * a
        assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * m
        assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * m
    else:
        T, info = run_dist(A, nranks, b, q, seed, oversample=p)
    assert np.all(np.tril(T, -1) == 0.0) and diag_blocks_ok(T, min(b, n), n)
    assert abs(np.linalg.norm(T) - np.linalg.norm(A)) <= 4 * m * EPS * np.linalg.norm(A)
    if selection_well_posed(A, min(b, n), q, seed, p, ref):
        par = check_parity(T, ref["T"], ref["a_fro"])
        assert par["diag_ok"] and par["ek_ok"], par


@pytest.mark.parametrize("m,n,b,nranks", [(188, 166, 16, 3), (188, 166, 16, 8), (700, 640, 32, 3), (300, 300, 8, 5)])
def test_dist_svd_chunk_slot_alignment(m, n, b, nranks):
    """Regression: a rank's deferred-SVD chunk starts at its own slot j0 =
    (steps < 8k it owns), odd for P = 3, 5, 8; the Jacobi work slice at j0
    must stay 16-byte aligned for the even-k vectorized block I/O (was a
    misaligned-address fault once a rank owned an odd number of steps before
    the second chunk)."""
    A = testmat.gaussian(m, n, 5)
    ref = oracle.randutv(A, b, 2, 9, build_ortho=False)
    T, info = run_dist(A, nranks, b, 2, 9)
    assert info.steps == ref["steps"] and info.steps > 8
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_dist_weak_scaling_shapes_loopback(nranks):
    """The exact matrices `bench.py --gpus N` factors at N = 2, 4, 8 (weak
    scaling: the c3 recipe at n = 10000 N^(1/3)), through the multi-GPU
    algorithm with N virtual ranks on one GPU: the same T diagonal as the
    single-GPU factorization (which test_gpu_fullsize pins to the oracle at
    full size) to rounding, exact triangularity and ||T||_F = ||A||_F."""
    At, c = testmat.device_config("c3", scale=nranks ** (1.0 / 3.0))
    A = At.t()
    m, n = A.shape
    comm = D.loopback(nranks)
    shards = [D.shard(A, c.b, r, nranks) for r in range(nranks)]
    Ts, info = D.factor(comm, shards, m, n, c.b, c.q, c.seed)
    torch.cuda.synchronize()
    comm.close()
    del shards
    T = D.assemble(Ts, n, c.b)
    del Ts
    assert info.k_done == n
    a = torch.linalg.norm(A).item()
    assert abs(torch.linalg.norm(T).item() - a) <= 4 * n * EPS * a
    assert not torch.any(torch.tril(T, -1) != 0).item()
    dd = torch.diagonal(T).abs().cpu().numpy()
    del T
    _, T1, _, _ = P.randutv(A, c.b, c.q, c.seed, with_uv=False)
    torch.cuda.synchronize()
    d1 = torch.diagonal(T1).abs().cpu().numpy()
    assert np.all(np.abs(d1 - dd) <= 1e-10 * d1 + n * EPS * a)


@pytest.mark.parametrize("m,n,b,q,nranks,uv", [(300, 500, 50, 1, 2, True), (400, 1000, 64, 1, 3, False),
                                               (130, 400, 32, 2, 4, True), (100, 333, 128, 1, 3, True),
                                               (256, 300, 50, 1, 5, False), (60, 700, 16, 1, 8, True)])
def test_dist_fat_parity(m, n, b, q, nranks, uv):
    """Fat inputs m < n (Remark "The case m < n", R8) through the multi-GPU
    algorithm: the final m_i x n_i block spans several ranks' columns; its
    transpose is allgathered and QR-factored on every rank, T(I1, J) and V are
    transformed through an allreduced r0 x m_i product.  T against the oracle's
    parity rule and the single-GPU fat path; with U, V the exact invariants."""
    A = testmat.gaussian(m, n, m + 3 * n + nranks)
    ref = oracle.randutv(A, b, q, 3, build_ortho=False)
    if uv:
        U, T, V, info = run_dist_uv(A, nranks, b, q, 3)
        a = np.linalg.norm(A)
        assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * n * a
        assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * n
        assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * n
    else:
        T, info = run_dist(A, nranks, b, q, 3)
    assert info.k_done == m
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par
    assert np.all(np.tril(T, -1) == 0.0)
    _, T1, _, _ = P.randutv(to_dev(A), b, q, 3, with_uv=False)
    d1, dd = np.abs(np.diag(T1.cpu().numpy())), np.abs(np.diag(T))
    assert np.all(np.abs(d1 - dd) <= 1e-10 * d1 + n * EPS * ref["a_fro"])


@pytest.mark.parametrize("m,n,b,q,nranks", [(1000, 1000, 64, 2, 4), (800, 600, 50, 1, 3), (640, 640, 64, 0, 2),
                                            (1500, 1200, 128, 2, 8)])
def test_dist_collectives_per_step(m, n, b, q, nranks):
    """Collectives of one distributed factorization (T-only, tol = 0, CholeskyQR
    path) against the per-step model of DESIGN.md §8: per randomized step
    2q + 3 allreduces (q re-orthonormalisation Grams, q Z = X Y, the QR(Y)
    Gram, the merged second Gram + top block of Q1, P = T W_v) and one
    broadcast (the panel's W_u, T_u, R11); one allreduce per SVD chunk of 8
    steps (its Us blocks for the row folds); two per call (||A||_F with the
    non-finite / aliasing flags, and the CholeskyQR verdict); no allgather."""
    A = testmat.gaussian(m, n, m + n)
    comm = D.loopback(nranks)
    Ad = to_dev(A)
    shards = [D.shard(Ad, b, r, nranks) for r in range(nranks)]
    Ts, info = D.factor(comm, shards, m, n, b, q, 3)
    torch.cuda.synchronize()
    st = comm.stats()
    comm.close()
    S = info.steps
    chunks = -(-S // 8)
    assert info.qr_fallbacks == 0
    assert st["allreduce"][0] == 2 + S * (2 * q + 3) + chunks, (st, S)
    assert st["bcast"][0] == S, st
    assert st["allgather"][0] == 0, st
    assert not st["aborted"]
    # payload of the per-step allreduces (bytes per rank), step i = 1..S
    per_step = sum(8 * (q * b * b + q * (m - b * (i - 1)) * b + b * b + 2 * b * b + m * b) for i in range(1, S + 1))
    assert st["allreduce"][1] == per_step + 8 * (3 + 1) + 8 * b * b * S, (st, per_step)
    T = D.assemble(Ts, n, b).cpu().numpy()
    ref = oracle.randutv(A, b, q, 3, build_ortho=False)
    par = check_parity(T, ref["T"], ref["a_fro"])
    assert par["diag_ok"] and par["ek_ok"], par


def test_dist_nccl_timeout_aborts():
    """NCCL failure handling: a host wait longer than RANDUTV_NCCL_TIMEOUT_S
    (here 0 s: the first wait that is not already complete) aborts the
    communicator (ncclCommAbort) and the call returns RANDUTV_ERR_NCCL; the
    aborted communicator then refuses further work with RANDUTV_ERR_NCCL."""
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(30200 + os.getpid() % 500)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    old = os.environ.get("RANDUTV_NCCL_TIMEOUT_S")
    os.environ["RANDUTV_NCCL_TIMEOUT_S"] = "0"
    try:
        comm = D.nccl_from_torch()
        c = testmat.config("c3", scale=0.2)
        with pytest.raises(P.RandUTVError) as e:
            D.factor(comm, [to_dev(c.A)], *c.A.shape, c.b, c.q, c.seed)
        assert e.value.code == 4                      # RANDUTV_ERR_NCCL
        assert comm.stats()["aborted"]
        with pytest.raises(P.RandUTVError) as e2:
            D.factor(comm, [to_dev(c.A)], *c.A.shape, c.b, c.q, c.seed)
        assert e2.value.code == 4
        comm.close()
    finally:
        if old is None:
            del os.environ["RANDUTV_NCCL_TIMEOUT_S"]
        else:
            os.environ["RANDUTV_NCCL_TIMEOUT_S"] = old
        torch.cuda.synchronize()
        dist.destroy_process_group()
