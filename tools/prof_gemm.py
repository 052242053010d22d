"""Run the three dominant c3 GEMM shapes once each (after warm-up) through the
C ABI, for an ncu capture:  ncu --set full -k regex:dgemm_kernel -s 6 -c 3 python tools/prof_gemm.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402

m = n = 10000
b = 256
X = P.empty_cm(m, n)
X.copy_(torch.randn(n, m, dtype=torch.float64, device="cuda").t())
G = torch.randn(b, m, dtype=torch.float64, device="cuda").t()
Y = P.empty_cm(n, b)
Z = P.empty_cm(m, b)
Wt = torch.randn(b, n, dtype=torch.float64, device="cuda").t()
shapes = [
    ("sketch Y = X^T G (TN)", lambda: P.dgemm(True, False, 1.0, X, G, 0.0, Y)),
    ("Z = X Y (NN)", lambda: P.dgemm(False, False, 1.0, X, Y, 0.0, Z)),
    ("update X -= Z W^T (NT)", lambda: P.dgemm(False, True, -1.0, Z, Wt, 1.0, X)),
]
for rep in range(3):
    for name, f in shapes:
        f()
torch.cuda.synchronize()
for name, f in shapes:
    f()
torch.cuda.synchronize()
print("done")
