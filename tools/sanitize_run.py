"""Small workload for compute-sanitizer (SURVEY §4 "Sanitizers"): config 1 and
a 1000^2 case through every kernel family (CholeskyQR2 + reconstruction,
Householder fallback, Jacobi, GEMM incl. split-K, U/V formation, loopback
multi-GPU).  usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from paper_1703_00998_b200 import dist as D  # noqa: E402


def dev(A):
    return torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()


c = testmat.config("c1")
U, T, V, info = P.randutv(dev(c.A), c.b, c.q, c.seed)                       # a1-a11 with U, V
A2 = testmat.gaussian(1000, 1000, 5)
_, T2, _, _ = P.randutv(dev(A2), 128, 1, 3, with_uv=False)                  # T-only, 7 steps
_, T3, _, _ = P.randutv(dev(A2), 128, 1, 3, with_uv=False, qr_mode=1)       # Householder panels
Vq, R, tau, Tw, fb = P.panel_qr(dev(testmat.gaussian(700, 64, 2)), mode=0, return_fallback=True)
comm = D.loopback(2)
sh = [D.shard(dev(A2), 128, r, 2) for r in range(2)]
Us, Ts, Vs, _ = D.factor(comm, sh, 1000, 1000, 128, 1, 3, with_uv=True)
torch.cuda.synchronize()
comm.close()
print("sanitize workload done", info.steps, float(T2.abs().max()), fb)
