"""Pins for oracle/philox.py (PAPER.md:941 ``randn``; reading R2)."""
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest
import scipy.stats

from oracle import philox

CURAND_HOST = r"""
#define QUALIFIERS static inline
#include <cstdio>
#include <vector_types.h>
#include <curand_philox4x32_x.h>
int main() {
  unsigned a[6];
  while (scanf("%u %u %u %u %u %u", &a[0], &a[1], &a[2], &a[3], &a[4], &a[5]) == 6) {
    uint4 c; c.x = a[0]; c.y = a[1]; c.z = a[2]; c.w = a[3];
    uint2 k; k.x = a[4]; k.y = a[5];
    uint4 r = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
}
"""


def _cuda_include():
    for d in ("/usr/local/cuda/include", "/usr/local/cuda-12.9/include"):
        if os.path.exists(os.path.join(d, "curand_philox4x32_x.h")):
            return d
    return None


@pytest.mark.skipif(_cuda_include() is None or shutil.which("g++") is None, reason="no cuRAND header / g++")
def test_philox_matches_curand_host():
    """Library pin: cuRAND's curand_Philox4x32_10 compiled for the host."""
    rng = np.random.default_rng(7)
    ctr = rng.integers(0, 2**32, size=(4, 64), dtype=np.uint64).astype(np.uint32)
    ctr[:, 0] = 0
    ctr[:, 1] = 0xFFFFFFFF
    keys = rng.integers(0, 2**32, size=(64, 2), dtype=np.uint64).astype(np.uint32)
    keys[0] = 0
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "t.cpp"), os.path.join(d, "t")
        open(src, "w").write(CURAND_HOST)
        subprocess.check_call(["g++", "-O1", "-I", _cuda_include(), src, "-o", exe])
        inp = "\n".join(" ".join(str(int(v)) for v in list(ctr[:, j]) + list(keys[j])) for j in range(64))
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout
    ref = np.array([[int(t) for t in line.split()] for line in out.strip().splitlines()], dtype=np.uint64)
    got = np.stack([philox.philox4x32_10(ctr[:, j:j + 1], keys[j])[:, 0] for j in range(64)]).astype(np.uint64)
    np.testing.assert_array_equal(got, ref)


def test_uniform_map_exact():
    """u = (2k+1) 2^-53 with k the top 52 bits: exact, odd multiple of 2^-53, in (0,1)."""
    w = np.array([[0, 0xFFFFFFFF, 0x12345678, 0], [0, 0xFFFFFFFF, 0x9ABCDEF0, 0x80000000],
                  [0, 0xFFFFFFFF, 1, 0], [0, 0xFFFFFFFF, 0, 0]], dtype=np.uint32)
    u, u2 = philox.uniforms(w)
    assert u[0] == 2.0 ** -53 and u[1] == 1.0 - 2.0 ** -53
    k = (int(0x9ABCDEF0) << 32 | 0x12345678) >> 12
    assert u[2] == (2 * k + 1) * 2.0 ** -53
    assert u[3] == (2 * (1 << 51) + 1) * 2.0 ** -53  # w = 2^63 -> k = 2^51
    scaled = u * 2.0 ** 53
    assert np.all(scaled == np.round(scaled)) and np.all(np.mod(scaled, 2) == 1)
    assert np.all((u > 0) & (u < 1)) and np.all((u2 > 0) & (u2 < 1))


def test_box_muller_identity_and_layout():
    """g_{2p}^2 + g_{2p+1}^2 = -2 ln u for the same counter; odd row counts drop the last sin."""
    G = philox.gaussian_block(11, 3, 9, 4)
    assert G.shape == (9, 4) and G.flags.f_contiguous
    G10 = philox.gaussian_block(11, 3, 10, 4)
    np.testing.assert_array_equal(G, G10[:9])
    p = np.arange(5, dtype=np.uint32)
    for c in range(4):
        ctr = np.stack([p, np.full_like(p, c), np.full_like(p, 3), np.zeros_like(p)])
        u, _ = philox.uniforms(philox.philox4x32_10(ctr, philox.seed_key(11)))
        np.testing.assert_allclose(G10[0::2, c] ** 2 + G10[1::2, c] ** 2, -2 * np.log(u), rtol=1e-14)


def test_gaussian_distribution():
    G = philox.gaussian_block(0, 0, 100000, 2)
    x = G.ravel()
    assert abs(x.mean()) < 0.01 and abs(x.var() - 1) < 0.02
    assert scipy.stats.kstest(x, "norm").pvalue > 1e-3
    # different steps / seeds / columns are different streams
    assert not np.array_equal(philox.gaussian_block(0, 1, 64, 2), philox.gaussian_block(0, 0, 64, 2))
    assert not np.array_equal(philox.gaussian_block(1, 0, 64, 2), philox.gaussian_block(0, 0, 64, 2))
    g = philox.gaussian_block(0, 0, 64, 2)
    assert abs(np.corrcoef(g[:, 0], g[:, 1])[0, 1]) < 0.5
