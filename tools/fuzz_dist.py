"""Extended randomized parity run of the multi-GPU algorithm on loopback ranks
(up to 8 ranks, over-sampling, U/V, early stop, Householder panels) against the
oracle; usage (GPU box): python tools/fuzz_dist.py SEED N."""
import sys, os, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch, testmat, oracle
from paper_1703_00998_b200 import dist as D
from util import check_parity, selection_well_posed
def to_dev(A): return torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
fails = 0
t0 = time.time()
for case in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    n = int(rng.integers(50, 1000)); m = n + int(rng.integers(0, 400))
    fat = rng.random() < 0.3
    if fat:
        m = int(rng.integers(5, n))
    b = int(rng.choice([8, 15, 16, 31, 32, 48, 64, 100])); q = int(rng.integers(0, 3))
    P = int(rng.integers(1, 9)); p = 0 if fat else int(rng.choice([0, 0, 3, 8])); qm = int(rng.integers(0, 2)) if rng.random() < 0.2 else 0; ks = int(rng.choice([0, 0, 0, 3 * b])); uv = bool(rng.integers(0, 2))
    seed = int(rng.integers(0, 2**31)); A = testmat.gaussian(m, n, seed % 997)
    try:
        comm = D.loopback(P); Ad = to_dev(A); sh = [D.shard(Ad, b, r, P) for r in range(P)]
        res = D.factor(comm, sh, m, n, b, q, seed, oversample=p, with_uv=uv, qr_mode=qm, k_stop=ks); torch.cuda.synchronize(); comm.close()
        bb = min(b, n)
        if uv:
            Us, Ts, Vs, info = res
            U = D.assemble(Us, m, bb).cpu().numpy(); T = D.assemble(Ts, n, bb).cpu().numpy(); V = D.assemble(Vs, n, bb).cpu().numpy()
            a = np.linalg.norm(A)
            mx = max(m, n)
            ok_uv = (np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * mx * a and np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * mx
                     and np.abs(V.T @ V - np.eye(n)).max() <= 1e-13 * mx)
        else:
            Ts, info = res; T = D.assemble(Ts, n, bb).cpu().numpy(); ok_uv = True
        ref = oracle.randutv(A, bb, q, seed, build_ortho=False, p=p, k_stop=ks)
        par = check_parity(T, ref["T"], ref["a_fro"])
        wp = selection_well_posed(A, bb, q, seed, p, ref, k_stop=ks)
        ok = (not wp or (par["diag_ok"] and par["ek_ok"])) and ok_uv and np.all(np.tril(T[:, :info.k_done], -1) == 0) \
            and abs(np.linalg.norm(T) - np.linalg.norm(A)) <= 4 * max(m, n) * 2.2e-16 * np.linalg.norm(A)
    except Exception as e:
        ok = False; par = str(e)
    if not ok:
        fails += 1
        print("FAIL", dict(m=m, n=n, b=b, q=q, P=P, p=p, uv=uv, seed=seed, qm=qm, ks=ks), par, flush=True)
print("cases done, fails:", fails, "time", round(time.time() - t0, 1), flush=True)
