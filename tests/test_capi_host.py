"""Host-side checks of the C ABI (no GPU): librexi.so loads, exports every function that
include/rexi.h declares, and its host-only planner entries (S0 of SURVEY.md 8(a)) agree with
the independent oracle and the paper."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, read_appendix_a
from oracle import coeffs as C


@pytest.fixture(scope="module")
def rexi():
    from paper_2008_11607_b200 import build
    build.build()
    from paper_2008_11607_b200 import rexi as R
    return R


def header_functions():
    src = open(os.path.join(ROOT, "include", "rexi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rexi_[A-Za-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(rexi):
    names = header_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(rexi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    # and the binding declares a prototype for each one
    assert set(names) == set(rexi.EXPORTS), set(names) ^ set(rexi.EXPORTS)


def test_abi_version(rexi):
    assert rexi.abi_version() == 1


def test_appendix_a_compiled_table_matches_golden(rexi):
    mu, rows = read_appendix_a()
    lmu, a = rexi.appendix_a()
    assert lmu == float(mu)
    assert len(a) == len(rows) == 25
    for (l, re_, im_), al in zip(rows, a):
        assert al.real == float(re_) and al.imag == float(im_), l


@pytest.mark.parametrize("h,M", [(0.5, 22), (0.5, 65), (1.0, 38), (0.1, 278), (0.5, 1149),
                                 (0.2, 150), (0.5, 4558), (0.3, 2000)])
def test_planner_terms_match_oracle(rexi, h, M):
    """S0 parity: the planner's alpha_n, C_{1,n}, C_{2,n}, Gamma_n (C++ long double) vs the
    oracle's (numpy longdouble), two independent implementations of PAPER.md:201-282, 321."""
    al, c1, c2, g = rexi.terms_host(h, M)
    n, oal, oc1, oc2, og = C.rexii_terms(h, M).half()
    assert len(al) == len(oal) == M + 25
    assert np.array_equal(g, og)
    assert np.abs(al - oal).max() <= 1e-15 * np.abs(oal).max()
    scale = max(np.abs(oc1).max(), np.abs(oc2).max())
    assert np.abs(c1 - oc1).max() <= 2e-15 * scale
    assert np.abs(c2 - oc2).max() <= 2e-15 * scale


@pytest.mark.parametrize("D,tau,tol,h", [(512, 1.0, 1e-8, 0.5), (64, 0.02, 1e-12, 0.5),
                                         (1024, 0.1, 1e-12, 0.5), (4096, 1.0, 1e-12, 0.5),
                                         (128, 1.0, 0.0, 0.5), (128, 1.0, 0.0, 1.0),
                                         (128, -3.0, 1e-10, 0.3)])
def test_rule_M_matches_oracle(rexi, D, tau, tol, h):
    assert rexi.rule_M(D, tau, tol, h) == C.M_lrsw(D, tau, h, tol if tol > 0 else None)


def test_terms_host_rejects_bad_args(rexi):
    with pytest.raises(ValueError):
        rexi.terms_host(3.5, 50)
    with pytest.raises(ValueError):
        rexi.terms_host(0.5, 5)


@pytest.mark.parametrize("h,M", [(0.2, 150), (0.5, 65), (0.2, 1000)])
def test_planner_rexi_terms_match_oracle(rexi, h, M):
    """NEXT-1 table: beta^Re_n of the planner vs the oracle, n = 0..N."""
    al, beta, zero, g = rexi.terms_host(h, M, "rexi")
    t = C.rexi_terms(h, M)
    sel = t.n >= 0
    assert np.abs(al - t.alpha[sel]).max() <= 1e-15 * np.abs(al).max()
    assert np.abs(beta - t.beta_re[sel]).max() <= 2e-15 * np.abs(t.beta_re).max()
    assert np.all(zero == 0)
    assert g[0] == 1.0 and np.all(g[1:] == 2.0)


@pytest.mark.parametrize("tol", [0.0, 1e-3, 1e-6, 1e-8, 1e-12, 1e-15])
def test_h_for_tol_matches_oracle(rexi, tol):
    assert rexi.h_for_tol(tol) == C.h_for_tol(tol)


def test_planner_refit_meets_paper_bound(rexi):
    """NEXT-2: the planner's extended-precision refit, evaluated by the oracle in 30-digit
    arithmetic, meets the paper's stated fit error (< 8e-15), and its REXII
    reproduces e^{ix} at the Fig. 1 threshold M = ceil(x/h) + 11."""
    mpmath = pytest.importorskip("mpmath")
    mu, a, defect = rexi.fit_gaussian(24, -5.133333333333333)
    assert defect < 8e-15
    mpmath.mp.dps = 30
    full = [complex(np.conj(v)) for v in a[:0:-1]] + [complex(v) for v in a]
    worst = 0.0
    for x in np.linspace(0.0, 30.0, 601):
        xm = mpmath.mpf(float(x))
        s_ = mpmath.mpc(0)
        for j, l in enumerate(range(-24, 25)):
            s_ += mpmath.mpc(full[j].real, full[j].imag) / (mpmath.mpc(0, 1) * xm + mpmath.mpf(mu) + mpmath.mpc(0, l))
        worst = max(worst, float(abs(s_.real - mpmath.exp(-xm * xm / 4) / mpmath.sqrt(4 * mpmath.pi))))
    assert worst < 8e-15
    # scalar REXII with the refit table (oracle evaluator, closed-form reference)
    h, X = 0.5, 30.0
    M = C.M_rule(X, h)
    t = C.rexii_terms(h, M, mu=mu, a=np.array(full))
    assert abs(C.rexii_scalar(X, h, M, t)[0] - np.exp(1j * X)) < 1e-13


def test_planner_refit_mu_scan(rexi):
    mu, a, defect = rexi.fit_gaussian(24, None)
    mu0, a0, d0 = rexi.fit_gaussian(24, -5.133333333333333)
    assert -7.0 <= mu <= -3.0 and defect <= d0 * 1.5
