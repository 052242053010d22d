"""Where the end-to-end (host-buffer) time of one config goes: H2D of A alone, the
device-buffer factorization (graph replay, and eager), D2H of T alone, and
randutv_factor on pinned host A, T.  Usage (GPU box): python tools/e2e_breakdown.py [c3]"""
import os, sys, time
sys.path.insert(0, ".")
import torch, testmat
import paper_1703_00998_b200 as P
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
dev = torch.device("cuda", 0)
At, case = testmat.device_config(name, device=dev, scale=1.0)
A = At.t(); m, n = A.shape
Ah = torch.empty(n, m, dtype=torch.float64, pin_memory=True); Ah.copy_(At)
Th = torch.empty(n, m, dtype=torch.float64, pin_memory=True)
D = torch.empty(n, m, dtype=torch.float64, device=dev)
def wall(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
h2d = wall(lambda: D.copy_(Ah, non_blocking=True))
d2h = wall(lambda: Th.copy_(D, non_blocking=True))
T = P.empty_cm(m, n, dev)
def fac(): P.randutv(A, case.b, case.q, case.seed, k_stop=case.k_stop, tol=case.tol, out=(None, T, None))
fac(); fac()
dev_ms = wall(fac)
def e2e():
    rc = P.factor_raw(m, n, Ah.data_ptr(), m, case.b, case.q, case.seed, case.k_stop, None, Th.data_ptr(), None)
    assert rc == 0
e2e_ms = wall(e2e, 3)
gb = m * n * 8 / 1e9
print(f"{name}: H2D {h2d:.2f} ms ({gb / h2d * 1e3:.1f} GB/s)  D2H {d2h:.2f} ms ({gb / d2h * 1e3:.1f} GB/s)  "
      f"device factorization {dev_ms:.2f} ms (RANDUTV_NO_GRAPH={os.environ.get('RANDUTV_NO_GRAPH', '0')})  "
      f"e2e {e2e_ms:.2f} ms  e2e - device - H2D = {e2e_ms - dev_ms - h2d:.2f} ms")
