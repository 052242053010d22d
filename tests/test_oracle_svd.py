"""Pins for oracle/small_svd.py."""
import json
import os

import numpy as np

from oracle.small_svd import small_svd

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_closed_forms():
    for case in json.load(open(os.path.join(GOLD, "small_svd_closed_forms.json")))["cases"]:
        R = np.array(case["R"])
        Us, D, Vs = small_svd(R)
        np.testing.assert_allclose(D, case["sigma"], rtol=1e-15)
        np.testing.assert_allclose(Us @ np.diag(D) @ Vs.T, R, atol=1e-15)


def test_random_triangular_graded():
    rng = np.random.default_rng(5)
    for b in (1, 7, 64):
        R = np.triu(rng.standard_normal((b, b))) @ np.diag(10.0 ** -np.linspace(0, 6, b))
        Us, D, Vs = small_svd(R)
        assert np.all(np.diff(D) <= 0) and np.all(D >= 0)
        assert np.linalg.norm(Us.T @ Us - np.eye(b)) < 1e-13 * b
        assert np.linalg.norm(Vs.T @ Vs - np.eye(b)) < 1e-13 * b
        assert np.linalg.norm(Us @ np.diag(D) @ Vs.T - R) < 1e-14 * b * np.linalg.norm(R)
        # canonical sign: largest |entry| of each Vs column is positive
        idx = np.argmax(np.abs(Vs), axis=0)
        assert np.all(Vs[idx, np.arange(b)] > 0)
