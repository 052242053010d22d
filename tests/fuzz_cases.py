"""The fixed random cases of the GPU fuzz test (tests/test_gpu_fuzz.py) and
their input generator, shared with the CPU test that checks the fuzz design
(tests/test_fuzz_design.py).  Seeds are fixed (reproducible)."""
import numpy as np


def make(rng, m, n, kind):
    A = rng.standard_normal((m, n))
    k = min(m, n)
    if kind == "graded":
        U, _ = np.linalg.qr(rng.standard_normal((m, k)))
        V, _ = np.linalg.qr(rng.standard_normal((n, k)))
        A = U @ np.diag(np.logspace(0, -rng.uniform(2, 10), k)) @ V.T
    elif kind == "lowrank":
        r = max(1, k // 3)
        A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) + 1e-9 * rng.standard_normal((m, n))
    return np.asfortranarray(A)


def effective(m, n, b, p):
    """(b, p) as the oracle sees them: b capped to min(m, n); p = 0 for fat
    inputs (over-sampling applies to m >= n, R8/R23) and capped so that b + p
    <= min(m, n)."""
    bb = min(b, m, n)
    if p > 0 and m < n:
        p = 0
    if p > 0:
        p = min(p, max(0, min(m, n) - bb))
    return bb, p


CASES = []
_rng = np.random.default_rng(20261020)
for _ in range(60):
    m = int(_rng.integers(3, 420))
    n = int(_rng.integers(3, 420))
    b = int(_rng.choice([1, 2, 7, 16, 31, 48, 64, 100, 500]))
    q = int(_rng.integers(0, 4))
    kind = str(_rng.choice(["gauss", "graded", "lowrank"]))
    qr_mode = int(_rng.integers(0, 2))
    p = int(_rng.choice([0, 0, 0, 3]))
    k_stop = int(_rng.choice([0, 0, 0, b * 2]))
    seed = int(_rng.integers(0, 2**31))
    if p > 0:
        # over-sampling (R23) selects the b dominant directions of a (b + p)-column
        # sketch: determined only when the spectrum separates them, so these
        # cases get graded spectra (a Gaussian's flat trailing spectrum leaves
        # the selection to rounding: valid but not comparable)
        kind = "graded"
    CASES.append((m, n, b, q, kind, qr_mode, p, k_stop, seed))

# dedicated over-sampling cases (m >= n, b + p < n; graded spectra, R23)
_rng = np.random.default_rng(20261021)
for _ in range(16):
    n = int(_rng.integers(24, 400))
    m = n + int(_rng.integers(0, 200))
    b = int(_rng.choice([2, 7, 16, 31, 48, 64]))
    b = min(b, n // 3)
    p = int(_rng.choice([1, 3, 8]))
    q = int(_rng.integers(0, 4))
    qr_mode = int(_rng.integers(0, 2))
    k_stop = int(_rng.choice([0, 0, b * 2]))
    seed = int(_rng.integers(0, 2**31))
    CASES.append((m, n, b, q, "graded", qr_mode, p, k_stop, seed))
