"""Isolated DMMA GEMM throughput on the exact per-step shapes of one c3
factorization (10000^2, b = 256, q = 2), per role, against the in-situ class
times of bench.py: how much of the GEMM time is shape (waves, tails) and how
much is interference between the concurrent streams.
usage: python tools/gemm_steps.py [n] [b] [q]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
q = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = n
X = P.empty_cm(m, n); X.normal_()
Wm = P.empty_cm(max(m, n), 2 * b); Wm.normal_()
Y = P.empty_cm(max(m, n), 2 * b)
Cm = P.empty_cm(m, n); Cm.normal_()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tot = {}
for i in range(1, n // b + 1):
    r0 = b * (i - 1)
    mi, ni = m - r0, n - r0
    if b * i >= min(m, n):
        break
    Xi = X[r0:, r0:]
    roles = {
        # sketch: Z = X Y (mi x b x ni), Y = X^T Z (ni x b x mi), q times each
        "sketch": [(False, False, Xi, Wm[:ni, :b], 0.0, Y[:mi, :b], q),
                   (True, False, Xi, Wm[:mi, :b], 0.0, Y[:ni, :b], q)],
        # right apply: P_big = T(:, J3) Q1 (m x b x ni-b), trailing update T(:, J3) -= P2 W^T (m x ni-b x b)
        "right": [(False, False, Cm[:, r0 + b:], Wm[:ni - b, :b], 0.0, Y[:m, :b], 1),
                  (False, True, Y[:m, :b], Wm[:ni - b, :b], 1.0, Cm[:, r0 + b:], 1)],
        # left apply: C^T [W_u | G''] (ni-b x 2b x mi), C -= WT (C^T W_u)^T (mi x ni-b x b)
        "left": [(True, False, Cm[r0:, r0 + b:], Wm[:mi, :2 * b], 0.0, Y[:ni - b, :2 * b], 1),
                 (False, True, Wm[:mi, :b], Y[:ni - b, :b], 1.0, Cm[r0:, r0 + b:], 1)],
    }
    for role, lst in roles.items():
        for ta, tb, A, B, beta, C, cnt in lst:
            Mm = A.shape[1] if ta else A.shape[0]
            Kk = A.shape[0] if ta else A.shape[1]
            Nn = B.shape[0] if tb else B.shape[1]
            if Mm == 0 or Nn == 0 or Kk == 0:
                continue
            ms = timed(lambda: P.dgemm(ta, tb, 1.0, A, B, beta, C))
            f = 2.0 * Mm * Nn * Kk
            t = tot.setdefault(role, [0.0, 0.0])
            t[0] += cnt * ms
            t[1] += cnt * f
for role, (ms, f) in tot.items():
    print(f"{role:7s} isolated sum {ms:8.2f} ms  {f / ms / 1e9:6.2f} TF  ({f:.3e} flops)")
ms = sum(v[0] for v in tot.values())
f = sum(v[1] for v in tot.values())
print(f"all     isolated sum {ms:8.2f} ms  {f / ms / 1e9:6.2f} TF")
