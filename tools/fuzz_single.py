"""Extended randomized parity run of the single-GPU path (shapes up to 1500^2,
all options) against the oracle; usage (GPU box): python tools/fuzz_single.py SEED N.
Element parity where the over-sampled selection is well posed (tests/util.py)."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch, oracle
import paper_1703_00998_b200 as P
from util import check_parity, selection_well_posed
def to_dev(A): return torch.from_numpy(np.ascontiguousarray(np.asarray(A).T)).cuda().t()
def make(rng, m, n, kind):
    A = rng.standard_normal((m, n)); k = min(m, n)
    if kind == "graded":
        U, _ = np.linalg.qr(rng.standard_normal((m, k))); V, _ = np.linalg.qr(rng.standard_normal((n, k)))
        A = U @ np.diag(np.logspace(0, -rng.uniform(2, 10), k)) @ V.T
    return np.asfortranarray(A)
rng = np.random.default_rng(int(sys.argv[1])); N = int(sys.argv[2]); fails = 0; t0 = time.time()
for _ in range(N):
    m = int(rng.integers(3, 1500)); n = int(rng.integers(3, 1500))
    b = int(rng.choice([1, 3, 8, 16, 31, 64, 96, 128, 200, 256, 512])); q = int(rng.integers(0, 4))
    kind = str(rng.choice(["gauss", "graded"])); qm = int(rng.random() < 0.2)
    p = int(rng.choice([0, 0, 4, 10])) if m >= n else 0
    ks = int(rng.choice([0, 0, 0, 2 * b])); uv = bool(rng.integers(0, 2)); seed = int(rng.integers(0, 2**31))
    A = make(rng, m, n, kind); bb = min(b, m, n)
    if p > 0: p = min(p, max(0, min(m, n) - bb))
    if bb + p > 512: p = 0
    try:
        U, T, V, info = P.randutv(to_dev(A), b, q, seed, k_stop=ks, qr_mode=qm, oversample=p, with_uv=uv)
        torch.cuda.synchronize()
        T = T.cpu().numpy(); a = np.linalg.norm(A); ok = np.all(np.isfinite(T))
        if uv:
            U, V = U.cpu().numpy(), V.cpu().numpy()
            ok &= np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * max(m, n) * a
            ok &= np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * max(m, n) and np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * max(m, n)
        ok &= abs(np.linalg.norm(T) - a) <= 4 * max(m, n) * 2.2e-16 * a
        ref = oracle.randutv(A, bb, q, seed, k_stop=ks, build_ortho=False, p=p)
        ok &= info.k_done == ref["k"] and np.all(np.tril(T[:, :info.k_done], -1) == 0)
        par = check_parity(T, ref["T"], ref["a_fro"])
        if selection_well_posed(A, bb, q, seed, p, ref, k_stop=ks):
            ok &= par["diag_ok"] and par["ek_ok"]
    except Exception as e:
        ok = False; par = repr(e)
    if not ok:
        fails += 1; print("FAIL", dict(m=m, n=n, b=b, q=q, kind=kind, qm=qm, p=p, ks=ks, uv=uv, seed=seed), par, flush=True)
        try:  # which side is off: both |diag T| (sorted) against LAPACK's singular values
            k = min(m, n)
            if ks == 0 and bb >= k:
                sv = np.linalg.svd(A, compute_uv=False)
                dg_ = np.sort(np.abs(np.diag(T)[:k]))[::-1]; do_ = np.sort(np.abs(np.diag(ref["T"])[:k]))[::-1]
                print("   max|gpu - svd| %.3e  max|oracle - svd| %.3e  sigma_min %.3e  fallbacks %d"
                      % (np.abs(dg_ - sv).max(), np.abs(do_ - sv).max(), sv.min(), info.qr_fallbacks), flush=True)
        except Exception as e:  # noqa: BLE001
            print("   diag:", e)
print("cases", N, "fails", fails, "time", round(time.time() - t0, 1), flush=True)
