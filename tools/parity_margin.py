"""Parity margins (tests/util.check_parity's max relative |t_jj| and e_k
deviations from the oracle) on the scaled BASELINE configs -- to compare two
settings of an A/B switch, run once per setting (the switches are read once
per process).  usage: python tools/parity_margin.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from util import check_parity  # noqa: E402

for name, scale, q in [("c2", 0.2, 1), ("c2", 0.2, 2), ("c2", 0.1, 2), ("c3", 0.1, 2), ("c3", 0.2, 2), ("c1", 1.0, 1),
                       ("c4", 0.05, 1)]:
    c = testmat.config(name, scale=scale, q=q)
    A = c.A
    ref = oracle.randutv(A, c.b, c.q, c.seed, build_ortho=False)
    _, T, _, info = P.randutv(torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t(), c.b, c.q, c.seed, with_uv=False)
    torch.cuda.synchronize()
    par = check_parity(T.cpu().numpy(), ref["T"], ref["a_fro"])
    print(f"{name} scale {scale} q {q}: diag_max_rel {par['diag_max_rel']:.2e} ek_max_rel {par['ek_max_rel']:.2e} "
          f"ok {par['diag_ok'] and par['ek_ok']}", flush=True)
