"""Time the panel QR (randutv_panel_qr_ex) on its own, both algorithms.
usage: python tools/bench_qr.py [m b] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00998_b200 as P  # noqa: E402

shapes = [(int(sys.argv[i]), int(sys.argv[i + 1])) for i in range(1, len(sys.argv) - 1, 2)] or \
    [(10000, 256), (5000, 256), (2000, 256), (20000, 256), (30000, 512)]
for m, b in shapes:
    Y = torch.randn(b, m, dtype=torch.float64, device="cuda").t()
    for mode in (0, 1):
        for _ in range(3):
            P.panel_qr(Y, mode=mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        reps = 10
        for _ in range(reps):
            P.panel_qr(Y, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        P.profile_begin()
        P.panel_qr(Y, mode=mode)
        prof = P.profile_end()
        parts = {k: round(v["ms"], 3) for k, v in prof.items() if v["launches"]}
        nl = {k: v["launches"] for k, v in prof.items() if v["launches"]}
        print(f"m={m} b={b} mode={mode}: {ms:.3f} ms/QR  by_class_ms={parts} launches={nl}", flush=True)
