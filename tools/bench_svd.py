"""Time the batched Jacobi SVD (randutv_small_svd_batched).
usage: python tools/bench_svd.py [batch k] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402

args = [int(x) for x in sys.argv[1:]]
shapes = list(zip(args[0::2], args[1::2])) or [(39, 256), (23, 128), (4, 512), (1, 16)]
for batch, k in shapes:
    g = torch.Generator(device="cuda").manual_seed(k)
    R = torch.randn(batch, k, k, dtype=torch.float64, device="cuda", generator=g).triu()
    R = R * torch.logspace(0, -4, k, dtype=torch.float64, device="cuda")[None, None, :]
    P.small_svd_batched(R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    D, Us, Vs, sw = P.small_svd_batched(R)
    e1.record()
    torch.cuda.synchronize()
    rec = (Us @ torch.diag_embed(D) @ Vs.transpose(1, 2) - R).norm() / R.norm()
    s_ref = torch.linalg.svdvals(R)
    err = ((D - s_ref).abs() / s_ref[:, :1]).max().item()
    print(f"batch={batch} k={k}: {e0.elapsed_time(e1):.3f} ms  sweeps={sw.max().item()}  recon={rec.item():.2e} "
          f"sigma_err/sigma1={err:.2e}", flush=True)
