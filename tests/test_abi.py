"""The C-ABI library builds, loads and exports every symbol include/randutv.h
declares (no GPU needed: only argument validation runs here)."""
import ctypes
import os
import re

import pytest

import paper_1703_00998_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "randutv.h")).read()
    return sorted(set(re.findall(r"RANDUTV_API\s+[\w\s\*]+?\b(randutv_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = P.lib()
    names = header_functions()
    assert len(names) == 26, names
    assert sorted(P.EXPORTED) == names
    for name in names:
        assert hasattr(L, name), name


def test_version_and_strerror():
    L = P.lib()
    assert b"sm_100a" in L.randutv_version()
    for code in (0, 1, 2, 3, 4, 5, -3):
        assert L.randutv_strerror(code)


def test_workspace_size_monotone():
    a = P.workspace_size(1000, 1000, 64, 1, False)
    b = P.workspace_size(1000, 1000, 64, 1, True)
    c = P.workspace_size(2000, 2000, 64, 1, False)
    assert 0 < a < b and a < c


@pytest.mark.parametrize("args,code", [
    (dict(m=0), -1), (dict(n=0), -2), (dict(A=None), -3), (dict(lda=3), -4),
    (dict(b=0), -5), (dict(b=2000), -5), (dict(q=-1), -6), (dict(k_stop=-1), -8),
    (dict(U=None), -9), (dict(T=None), -10),
])
def test_argument_errors(args, code):
    buf = (ctypes.c_double * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p).value
    kw = dict(m=5, n=4, A=p, lda=5, b=2, q=1, seed=0, k_stop=0, U=p, T=p, V=p)
    kw.update(args)
    rc = P.factor_raw(kw["m"], kw["n"], kw["A"], kw["lda"], kw["b"], kw["q"], kw["seed"], kw["k_stop"], kw["U"],
                      kw["T"], kw["V"])
    assert rc == code


def test_flop_formula_matches_paper_ratios():
    """randUTV/CPQR = 3, 4, 5 for q = 0, 1, 2 (m = n)."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "flop_ratios.json")))
    n = 1000
    for q, ratio in g["ratio_vs_cpqr_square"].items():
        assert abs(P.flops.flops_T(n, n, int(q)) / P.flops.flops_cpqr(n, n) - ratio) < 1e-12


def test_flop_step_sum_limit():
    """The per-step sum tends to the paper's formula."""
    for q in (0, 1, 2):
        f = P.flops.flops_T(10000, 10000, q)
        s = P.flops.flops_T_steps(10000, 10000, 256, q)
        assert 1.0 < s / f < 1.06
        s2 = P.flops.flops_T_steps(10000, 10000, 2, q)
        assert abs(s2 / f - 1) < 1e-3
