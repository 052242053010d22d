"""One warm-up + N profiled randUTV factorizations of a config (for ncu runs).
usage: python tools/prof_step.py [config] [steps] [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
At, c = testmat.device_config(name, scale=scale)
A = At.t()
m, n = A.shape
T = P.empty_cm(m, n)
P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None))
torch.cuda.synchronize()
l0 = P.launch_count()
for _ in range(steps):
    P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None))
torch.cuda.synchronize()
print(f"launches_per_step={(P.launch_count() - l0) // steps} warmup_launches={l0}")
