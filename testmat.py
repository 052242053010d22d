"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NO arithmetic of the randUTV method (no sketching, no
Householder, no SVD of the method): only the recipes that build the input
matrices A of BASELINE.json's five configurations.  Neither ``oracle/`` nor the
CUDA package imports it; both are *fed* from it.

Recipes (BASELINE.json ``configs``):

* c1: 500x500 i.i.d. N(0,1), seed 0.
* c2: 3000x3000 = Q1 diag(sigma) Q2^T, sigma_j = 10^(-12 (j-1)/(n-1)),
  Q1, Q2 Haar (QR of a Gaussian, sign-fixed so that diag R > 0).
* c3: 10000x10000 = Q1 diag(sigma) Q2^T with the S-shaped spectrum
  sigma_j = 1 (j <= 2000), 10^(-8 (j-2000)/1000) (2000 < j <= 3000),
  1e-8 (j > 3000)  (BASELINE governs over PAPER.md:1424-1428).
* c4: 20000x8000 i.i.d. N(0,1).
* c5: 30000x30000 = X Y^T + 1e-8 N(0,1), X, Y 30000x2000 i.i.d. N(0,1).

The paper's matrices (§6.2) are of the same families;
no public dataset is involved.  The ``scale`` argument shrinks a recipe
proportionally (breakpoints scale with n) for CPU-sized parity cases.

All host matrices are returned as column-major (Fortran-ordered) float64
numpy arrays; device matrices as torch tensors whose *transpose view* is the
column-major matrix (see ``paper_1703_00998_b200.as_colmajor``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


# --------------------------------------------------------------------------- spectra
def sigma_exponential(n: int, decades: float = 12.0) -> np.ndarray:
    """sigma_j = 10^(-decades (j-1)/(n-1)), j = 1..n (config 2)."""
    j = np.arange(n, dtype=np.float64)
    return 10.0 ** (-decades * j / max(n - 1, 1))


def sigma_s_shape(n: int, flat: int, drop_end: int, floor_decades: float = 8.0) -> np.ndarray:
    """S-shaped spectrum (config 3): 1 for j <= flat, log-linear drop to
    10^-floor_decades over flat < j <= drop_end, then constant."""
    j = np.arange(1, n + 1, dtype=np.float64)
    s = np.ones(n)
    mid = (j > flat) & (j <= drop_end)
    s[mid] = 10.0 ** (-floor_decades * (j[mid] - flat) / float(drop_end - flat))
    s[j > drop_end] = 10.0 ** (-floor_decades)
    return s


# --------------------------------------------------------------------------- host generators
def gaussian(m: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    # draw n x m row-major == m x n column-major, no copy
    return rng.standard_normal((n, m)).T


def haar(n: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-distributed orthogonal matrix: QR of a Gaussian, Q <- Q diag(sign(diag R))."""
    g = rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d[None, :]


def with_spectrum(m: int, n: int, sigma: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q1 = haar(m, rng)[:, : len(sigma)]
    q2 = haar(n, rng)[:, : len(sigma)]
    return np.asfortranarray((q1 * sigma[None, :]) @ q2.T)


def low_rank_plus_noise(n: int, rank: int, noise: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, rank))
    y = rng.standard_normal((n, rank))
    return np.asfortranarray(x @ y.T + noise * rng.standard_normal((n, n)))


@dataclass
class Case:
    """One factorization problem: A plus the method's parameters."""
    name: str
    A: np.ndarray
    b: int
    q: int
    seed: int
    k_stop: int = 0
    tol: float = 0.0
    sigma: np.ndarray | None = None  # known singular values when analytic
    meta: dict = field(default_factory=dict)


SEEDS = {"c1": 0, "c2": 2, "c3": 3, "c4": 4, "c5": 5}


def config(name: str, scale: float = 1.0, q: int | None = None, build_A: bool = True) -> Case:
    """BASELINE.json config ``name`` ('c1'..'c5'); ``scale`` < 1 shrinks it
    (n -> round(n*scale), b kept unless it would exceed n/4).  ``build_A`` =
    False returns the parameters only (A = None)."""
    seed = SEEDS[name]
    mk = (lambda f, *a: f(*a)) if build_A else (lambda f, *a: None)
    if name == "c1":
        n = max(8, round(500 * scale))
        b = min(50, max(2, n // 4))
        return Case("c1", mk(gaussian, n, n, seed), b, 1 if q is None else q, seed)
    if name == "c2":
        n = max(8, round(3000 * scale))
        b = min(128, max(2, n // 4))
        s = sigma_exponential(n)
        return Case("c2", mk(with_spectrum, n, n, s, seed), b, 2 if q is None else q, seed, sigma=s)
    if name == "c3":
        n = max(16, round(10000 * scale))
        b = min(256, max(2, n // 8))
        s = sigma_s_shape(n, round(0.2 * n), round(0.3 * n))
        return Case("c3", mk(with_spectrum, n, n, s, seed), b, 2 if q is None else q, seed, sigma=s)
    if name == "c4":
        m, n = max(16, round(20000 * scale)), max(8, round(8000 * scale))
        b = min(256, max(2, n // 8))
        return Case("c4", mk(gaussian, m, n, seed), b, 1 if q is None else q, seed)
    if name == "c5":
        n = max(32, round(30000 * scale))
        rank = max(2, round(2000 * scale))
        b = min(512, max(2, n // 16))
        k_stop = max(b, round(2048 * scale))
        return Case("c5", mk(low_rank_plus_noise, n, rank, 1e-8, seed), b, 1 if q is None else q, seed,
                    k_stop=k_stop, tol=1e-6, meta={"rank": rank})
    raise KeyError(name)


# --------------------------------------------------------------------------- pinned host inputs
# OpenBLAS results depend on the kernel family it picks for the CPU and on its
# thread count (both change the summation order of dgemm / dgeqrf).  The
# recipes that go through LAPACK/BLAS (c2, c3: Haar QRs and the product; c5:
# X Y^T) are therefore run in a child process with both pinned, so the bytes
# of A are the same on every x86-64 host with AVX2 -- the full-size golden
# oracle values in tests/golden/ are keyed by the SHA-256 of those bytes.
PINNED_BLAS_ENV = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "8", "OMP_NUM_THREADS": "8"}


def sha256_colmajor(A: np.ndarray) -> str:
    import hashlib
    return hashlib.sha256(np.asfortranarray(A).tobytes(order="F")).hexdigest()


def config_pinned(name: str, scale: float = 1.0, q: int | None = None, tmpdir: str | None = None) -> Case:
    """:func:`config` with A built in a child process under ``PINNED_BLAS_ENV``
    (bit-reproducible across hosts); ``case.meta['sha256']`` = SHA-256 of A's
    column-major bytes."""
    import os
    import subprocess
    import sys
    import tempfile

    import shutil

    c = config(name, scale, q, build_A=False)
    if name == "c4":
        need = 8.8 * max(16, round(20000 * scale)) * max(8, round(8000 * scale))
    else:
        need = 8.8 * max(16, round({"c1": 500, "c2": 3000, "c3": 10000, "c5": 30000}[name] * scale)) ** 2
    d = tmpdir
    if d is None:  # /dev/shm when it has room (container defaults can be 64 MB), else the temp dir
        d = "/dev/shm" if os.path.isdir("/dev/shm") and shutil.disk_usage("/dev/shm").free > need else None
    fd, path = tempfile.mkstemp(suffix=".f64", dir=d)
    os.close(fd)
    try:
        here = os.path.dirname(os.path.abspath(__file__))
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import testmat; "
                "c = testmat.config(%r, %r, build_A=True); "
                "np.asfortranarray(c.A).T.tofile(%r); print(c.A.shape[0], c.A.shape[1])" % (here, name, scale, path))
        env = dict(os.environ, **PINNED_BLAS_ENV)
        out = subprocess.run([sys.executable, "-c", code], env=env, check=True, capture_output=True, text=True)
        m, n = (int(v) for v in out.stdout.split())
        A = np.fromfile(path, dtype=np.float64).reshape(n, m).T   # column-major m x n, no copy
    finally:
        os.unlink(path)
    c.A = A
    c.meta["sha256"] = sha256_colmajor(A)
    return c


# --------------------------------------------------------------------------- device generators
def device_config(name: str, device="cuda", scale: float = 1.0):
    """Full-size configs generated on the GPU with torch (harness only; the
    product never calls this).  Returns (A_colmajor_tensor_T, Case-without-A).
    The returned tensor ``At`` is n x m row-major, i.e. A = At.T is m x n
    column-major.  Same recipes as :func:`config`, different random stream."""
    import torch

    seed = SEEDS[name]
    g = torch.Generator(device=device)
    g.manual_seed(1000 + seed)
    f64 = torch.float64

    def randn(r, c):
        return torch.randn(r, c, generator=g, device=device, dtype=f64)

    def haar_t(n):
        qm, rm = torch.linalg.qr(randn(n, n))
        d = torch.sign(torch.diagonal(rm))
        d[d == 0] = 1
        return qm * d[None, :]

    if name in ("c1", "c4"):
        if name == "c1":
            m = n = max(8, round(500 * scale)); b, q = min(50, max(2, n // 4)), 1
        else:
            m, n = max(16, round(20000 * scale)), max(8, round(8000 * scale)); b, q = min(256, max(2, n // 8)), 1
        At = randn(n, m)
        return At, Case(name, None, b, q, seed)
    if name in ("c2", "c3"):
        if name == "c2":
            n = max(8, round(3000 * scale)); b, q = min(128, max(2, n // 4)), 2
            s = sigma_exponential(n)
        else:
            n = max(16, round(10000 * scale)); b, q = min(256, max(2, n // 8)), 2
            s = sigma_s_shape(n, round(0.2 * n), round(0.3 * n))
        q1, q2 = haar_t(n), haar_t(n)
        st = torch.tensor(s, device=device, dtype=f64)
        A = (q1 * st[None, :]) @ q2.T          # m x n, row-major storage
        At = A.T.contiguous()                   # column-major storage of A
        del q1, q2, A
        return At, Case(name, None, b, q, seed, sigma=s)
    if name == "c5":
        n = max(32, round(30000 * scale)); rank = max(2, round(2000 * scale))
        b = min(512, max(2, n // 16)); k_stop = max(b, round(2048 * scale))
        X, Y = randn(n, rank), randn(n, rank)
        At = (Y @ X.T)                          # (X Y^T)^T stored row-major = X Y^T column-major
        At.add_(randn(n, n), alpha=1e-8)
        return At, Case(name, None, b, 1, seed, k_stop=k_stop, tol=1e-6, meta={"rank": rank})
    raise KeyError(name)
