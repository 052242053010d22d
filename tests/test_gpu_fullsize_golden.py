"""Whole-factorization parity at BASELINE.json's full sizes for c3, c4 and c5
(Fig. fig:randUTV; the tall 12064 x 64 final block of c4,
P:896-903 / P:970-978; the early stop of c5), in the
configuration bench.py times (T-only, device buffers).

The oracle's values come from ``tests/golden/fullsize_<cfg>.npz``, written by
``tools/gen_golden_fullsize.py`` -- a committed script that calls only
``oracle/`` on the host matrix of ``testmat.config_pinned`` (BLAS-pinned, so its
bytes are the same on every x86-64 host; the file stores their SHA-256).  This
test builds the same host matrix, checks the hash, factors those exact bytes on
the GPU and compares EVERY |t_jj| and EVERY e_k = ||T(k+1:m, :)||_F under rule
R18: |diag| within 1e-10 relative and e_k within 1e-8 relative,
each plus the rounding floor F = max(m, n) eps ||A||_F.  Should the host bytes
differ (a BLAS that ignores the pinning), the oracle is run live on them
instead (minutes), so the comparison is always on identical inputs.
"""
import json
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_1703_00998_b200 as P  # noqa: E402
import testmat  # noqa: E402
from util import EPS, diag_blocks_ok, ek_fro  # noqa: E402

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"fullsize_{name}.npz"))
    return json.loads(str(z["meta"])), z["diag"], z["ek"]


def reference_values(name, c):
    """(meta, |diag T|, e_k) of the oracle on exactly c.A's bytes."""
    meta, diag, ek = load_golden(name)
    if c.meta["sha256"] == meta["sha256"]:
        return meta, diag, ek, "golden"
    t = time.time()
    ref = oracle.randutv(c.A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, build_ortho=False)
    T = ref["T"]
    live = dict(meta, steps=ref["steps"], k=ref["k"], a_fro=ref["a_fro"], trailing_fro=ref["trailing_fro"],
                oracle_seconds=round(time.time() - t, 1))
    return live, np.abs(np.diag(T))[: min(T.shape)], ek_fro(T), "live"


def gpu_values(c):
    m, n = c.A.shape
    At = torch.from_numpy(np.ascontiguousarray(c.A.T)).cuda()   # (n, m) row-major = A column-major
    A = At.t()
    T = P.empty_cm(m, n)
    _, T, _, info = P.randutv(A, c.b, c.q, c.seed, k_stop=c.k_stop, tol=c.tol, with_uv=False, out=(None, T, None))
    torch.cuda.synchronize()
    diag = torch.diagonal(T).abs().cpu().numpy()
    r2 = (T * T).sum(dim=1)                                      # row norms^2, fp64 on the GPU
    tail = torch.flip(torch.cumsum(torch.flip(r2, [0]), 0), [0])
    ek = torch.sqrt(torch.cat([tail, tail.new_zeros(1)])[: n + 1]).cpu().numpy()
    a_fro = torch.linalg.norm(A).item()
    k = info.k_done
    tril_nz = torch.count_nonzero(torch.tril(T[:, :k], -1)).item()
    blocks_ok = diag_blocks_ok(T[:k, :k].cpu().numpy(), c.b, k)
    del At, A, T, r2, tail
    torch.cuda.empty_cache()
    return info, diag, ek, a_fro, tril_nz, blocks_ok


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_fullsize_whole_factorization_vs_oracle(name):
    c = testmat.config_pinned(name)
    meta, d_ref, e_ref, src = reference_values(name, c)
    m, n = c.A.shape
    assert meta["shape"] == [m, n] and meta["b"] == c.b and meta["q"] == c.q and meta["seed"] == c.seed
    info, d_gpu, e_gpu, a_fro, tril_nz, blocks_ok = gpu_values(c)
    # the same stopping point and structure as the oracle
    assert info.steps == meta["steps"] and info.k_done == meta["k"], (info.steps, info.k_done, meta)
    assert tril_nz == 0 and blocks_ok
    assert abs(a_fro - meta["a_fro"]) <= 4 * max(m, n) * EPS * meta["a_fro"]
    F = max(m, n) * EPS * meta["a_fro"]                          # R18 rounding floor
    k = meta["k"]
    # every |t_jj| of the processed columns (1e-10 relative + F)
    dd = np.abs(d_gpu[:k] - d_ref[:k])
    bad_d = dd > 1e-10 * d_ref[:k] + F
    # every rank-k error e_k, k = 0..n (1e-8 relative + F)
    de = np.abs(e_gpu - e_ref)
    bad_e = de > 1e-8 * e_ref + F
    rel_d = float(np.max(dd / np.maximum(d_ref[:k], F)))
    rel_e = float(np.max(de / np.maximum(e_ref, F)))
    print(f"{name} [{src}]: steps={info.steps} k={k} max |diag| dev {rel_d:.2e} (rel, floored), "
          f"max e_k dev {rel_e:.2e}; {int(bad_d.sum())} / {int(bad_e.sum())} outside R18")
    assert not bad_d.any(), (int(bad_d.sum()), rel_d, np.flatnonzero(bad_d)[:10])
    assert not bad_e.any(), (int(bad_e.sum()), rel_e, np.flatnonzero(bad_e)[:10])
    if k < min(m, n):                                            # early stop (c5): the trailing norm
        assert abs(info.trailing_fro - meta["trailing_fro"]) <= 1e-8 * meta["trailing_fro"] + F
