"""Our DMMA GEMM vs cuBLAS (torch fp64 matmul) on the randUTV shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402

def t_ours(ta, tb, M, N, K, beta=0.0):
    A = P.empty_cm(K, M) if ta else P.empty_cm(M, K)
    B = P.empty_cm(N, K) if tb else P.empty_cm(K, N)
    A.normal_(); B.normal_()
    C = P.empty_cm(M, N); C.zero_()
    for _ in range(2):
        P.dgemm(ta, tb, 1.0, A, B, beta, C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        P.dgemm(ta, tb, 1.0, A, B, beta, C)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    Cref = (A.t() if ta else A) @ (B.t() if tb else B)
    err = ((C - beta * 0 - Cref).abs().max() / Cref.abs().max()).item() if beta == 0 else 0.0
    e0.record()
    for _ in range(5):
        Cref = (A.t() if ta else A) @ (B.t() if tb else B)
    e1.record(); torch.cuda.synchronize()
    ms_ref = e0.elapsed_time(e1) / 5
    f = 2.0 * M * N * K
    return f / ms / 1e9, f / ms_ref / 1e9, err

for (ta, tb, M, N, K, beta, what) in [
        (True, False, 10000, 256, 10000, 0.0, "Y = X^T G (sketch, TN)"),
        (False, False, 10000, 256, 10000, 0.0, "Z = X Y (sketch / right P, NN)"),
        (False, True, 10000, 10000, 256, 1.0, "T -= P W^T (rank-b update, NT)"),
        (True, False, 5000, 256, 5000, 0.0, "TN half size"),
        (False, True, 5000, 5000, 256, 1.0, "NT half size"),
        (False, False, 10000, 256, 256, 0.0, "P T_v (NN, K=b)"),
        (True, False, 256, 16, 10000, 0.0, "panel-QR S^T (skinny)"),
        (False, False, 10000, 240, 16, 1.0, "panel-QR update (K=16)"),
]:
    ours, ref, err = t_ours(ta, tb, M, N, K, beta)
    print(f"{what:34s} {M}x{N}x{K}: ours {ours:6.2f} TF  cuBLAS {ref:6.2f} TF  relerr {err:.1e}", flush=True)
