"""A/B timing of the panel-QR mode (0 = CholeskyQR2 + reconstruction, 1 =
Householder) on the latency-bound configs, CUDA-event timed per factorization.
usage: python tools/ab_qrmode.py [config ...]   (env RANDUTV_NO_GRAPH=1: eager)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402

for name in (sys.argv[1:] or ["c1", "c2"]):
    At, c = testmat.device_config(name)
    A = At.t()
    m, n = A.shape
    T = P.empty_cm(m, n)
    res = {}
    for rep in range(2):
        for mode in (0, 1):
            for _ in range(3):
                P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None),
                          qr_mode=mode)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            s = torch.cuda.current_stream()
            e0.record(s)
            for _ in range(reps):
                P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None),
                          qr_mode=mode)
            e1.record(s)
            torch.cuda.synchronize()
            res.setdefault(mode, []).append(e0.elapsed_time(e1) / reps)
    print(name, {k: [round(x, 3) for x in v] for k, v in res.items()},
          "graph" if not os.environ.get("RANDUTV_NO_GRAPH") else "eager", flush=True)
