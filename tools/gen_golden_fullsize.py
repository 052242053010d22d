"""Write the full-size whole-factorization oracle values of BASELINE.json's
c3, c4 and c5 to tests/golden/fullsize_<cfg>.npz.

Calls only ``oracle/`` (and ``testmat`` for the input, built with the
BLAS-pinned recipe ``testmat.config_pinned`` so its bytes are reproducible on
any x86-64 host; the file stores their SHA-256).  Nothing here comes from the
CUDA path.  The values are those the GPU parity rule R18 compares:

* ``diag``  = |t_jj|, j = 1..min(m, n)        (|diag T|, 1e-10 relative + F)
* ``ek``    = e_k = ||T(k+1:m, :)||_F, k = 0..n (rank-k errors, 1e-8 relative + F)
* ``steps``, ``k`` (columns processed), ``a_fro``, ``trailing_fro``

The oracle is run as it stands (Fig. fig:randUTV; T-only,
the bench's mode; c5 with k_stop = 2048 and tol = 1e-6).

    python tools/gen_golden_fullsize.py c3 c4 c5      # ~ 5 / 5 / 15 min on 8 cores
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import testmat  # noqa: E402


def ek_fro(T):
    r2 = np.einsum("ij,ij->i", T, T)
    tail = np.concatenate([np.cumsum(r2[::-1])[::-1], [0.0]])
    return np.sqrt(tail[: T.shape[1] + 1])


def main(names):
    for name in names:
        t0 = time.time()
        c = testmat.config_pinned(name)
        t1 = time.time()
        ref = oracle.randutv(c.A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, build_ortho=False)
        t2 = time.time()
        T = ref["T"]
        k = min(T.shape)
        meta = {"config": name, "shape": list(c.A.shape), "b": c.b, "q": c.q, "seed": c.seed,
                "k_stop": c.k_stop, "tol": c.tol, "sha256": c.meta["sha256"],
                "blas_env": testmat.PINNED_BLAS_ENV, "steps": ref["steps"], "k": ref["k"],
                "a_fro": ref["a_fro"], "trailing_fro": ref["trailing_fro"],
                "oracle_seconds": round(t2 - t1, 1), "input_seconds": round(t1 - t0, 1),
                "cores": os.cpu_count(),
                "writer": "tools/gen_golden_fullsize.py (oracle/ only)"}
        out = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
        np.savez_compressed(out, diag=np.abs(np.diag(T))[:k], ek=ek_fro(T), meta=json.dumps(meta))
        print(json.dumps(meta), flush=True)
        del c, ref, T


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c4", "c5"])
