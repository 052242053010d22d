"""Print SHA-256 of the pinned host test matrices (testmat.config_pinned) to
check that the host input recipe is bitwise reproducible across machines (the
golden full-size oracle values in tests/golden/ are keyed by these hashes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import testmat  # noqa: E402

cases = [a.split(":") for a in sys.argv[1:]] or [["c2", "1.0"], ["c3", "0.3"], ["c5", "0.1"]]
for name, scale in cases:
    t = time.time()
    c = testmat.config_pinned(name, float(scale))
    print(f"{name} scale={scale} shape={c.A.shape} sha={c.meta['sha256'][:16]} t={time.time() - t:.1f}s", flush=True)
