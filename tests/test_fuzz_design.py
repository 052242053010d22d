"""CPU check of the GPU fuzz test's design (tests/fuzz_cases.py): at most a
quarter of its over-sampled cases may fall back to invariants-only, i.e. have a
selection of the sketch's b dominant directions that the oracle itself does
not reproduce under a 1e-15 relative perturbation of A (R23)."""
import numpy as np

import oracle
from fuzz_cases import CASES, effective, make
from util import selection_well_posed


def test_fuzz_oversampling_cases_mostly_well_posed():
    over = [c for c in CASES if effective(c[0], c[1], c[2], c[6])[1] > 0]
    assert len(over) >= 8
    gated = []
    for m, n, b, q, kind, qr_mode, p, k_stop, seed in over:
        bb, pp = effective(m, n, b, p)
        A = make(np.random.default_rng(seed), m, n, kind)
        ref = oracle.randutv(A, bb, q, seed, k_stop=k_stop, build_ortho=False, p=pp)
        if not selection_well_posed(A, bb, q, seed, pp, ref, k_stop=k_stop):
            gated.append((m, n, b, q, kind, p))
    print(f"over-sampled fuzz cases: {len(over)}, invariants-only: {len(gated)} {gated}")
    assert len(gated) <= len(over) // 4, gated
