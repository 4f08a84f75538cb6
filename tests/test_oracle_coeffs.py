"""Pins for the oracle's coefficient generation (oracle/coeffs.py) against what the
paper and mathematics fix: the printed table, closed forms (e^{ix}, psi), the
Fig. 1 thresholds, the Appendix B constants and the printed M values."""
import math

import numpy as np
import pytest

from conftest import read_appendix_a
from oracle import coeffs as C


def test_appendix_a_copy_matches_golden():
    mu, rows = read_appendix_a()
    assert C.MU_APPENDIX_A == mu
    assert len(rows) == len(C.A_APPENDIX_A) == 25
    for (l, re, im), (ore, oim) in zip(rows, C.A_APPENDIX_A):
        assert float(re) == float(ore) and float(im) == float(oim), l


def test_rational_fit_defect_fp64():
    """max-norm error of R vs psi_1 "less than 8e-15"; reading G11: the
    fp64 evaluation adds rounding, so the fp64 check uses 1e-14 on [-30, 30]."""
    x = np.linspace(-30, 30, 20001)
    assert np.abs(C.R_real_form(x) - C.psi(1.0, x)).max() < 1e-14
    assert np.abs(C.R_complex_form(x) - C.psi(1.0, x)).max() < 1e-14


def test_rational_fit_defect_exact_arithmetic():
    """Same claim in 30-digit arithmetic: < 8e-15 (G11 measured 4.92e-15)."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 30
    mu = mpmath.mpf(C.MU_APPENDIX_A)
    a = [mpmath.mpc(mpmath.mpf(r), mpmath.mpf(i)) for r, i in C.A_APPENDIX_A]
    worst = mpmath.mpf(0)
    for x in np.linspace(0.0, 30.0, 1201):   # R and psi are even
        xm = mpmath.mpf(float(x))
        s = mpmath.mpc(0)
        for l in range(-24, 25):
            al = a[l] if l >= 0 else mpmath.conj(a[-l])
            s += al / (mpmath.mpc(0, 1) * xm + mu + mpmath.mpc(0, l))
        d = abs(s.real - mpmath.exp(-xm * xm / 4) / mpmath.sqrt(4 * mpmath.pi))
        worst = max(worst, d)
    assert worst < 8e-15
    assert worst > 1e-16   # a genuine fit, not an identity


def test_sign_reading_G1_discriminates():
    """The other reading of the sign column (sign on the whole number) is not a fit."""
    mu, a, L = C.appendix_a()
    a_alt = a.copy()
    for l in range(0, L + 1):
        re, im = C.A_APPENDIX_A[l]
        if float(re) < 0:   # printed '-' -> negate the whole printed number
            z = -(abs(float(re)) + 1j * float(im))
            a_alt[L + l] = z
            a_alt[L - l] = np.conj(z)
    x = np.linspace(-30, 30, 2001)
    assert np.abs(C.R_complex_form(x, mu, a_alt) - C.psi(1.0, x)).max() > 1.0


def test_real_and_complex_forms_agree():
    """eq:A(x,mu) is the real form of eq:ratapproxgaush1 when a_{-l} = conj(a_l)."""
    x = np.linspace(-50, 50, 5001)
    assert np.abs(C.R_real_form(x) - C.R_complex_form(x)).max() < 2e-16 * 300


def test_bm_closed_form():
    """eq:bm: |b_m| = e^{h^2}, b_0 = e^{h^2}, conj(b_m) = b_{-m}."""
    h, M = 0.5, 40
    re, im = C.b_coeffs_ld(h, M)
    b = re.astype(float) + 1j * im.astype(float)
    assert abs(b[M] - math.exp(h * h)) < 1e-15
    assert np.allclose(np.abs(b), math.exp(h * h), rtol=1e-15, atol=0)
    assert np.allclose(np.conj(b), b[::-1], rtol=0, atol=1e-15)
    assert abs(b[M + 1] - math.exp(0.25) * (math.cos(0.5) - 1j * math.sin(0.5))) < 1e-15
    with pytest.raises(ValueError):
        C.b_coeffs_ld(math.pi, 3)


def test_gaussian_sum_step1():
    """eq:eixsumM with eq:Mformula: accurate iff |x| <= (M-11)h."""
    assert abs(C.gaussian_sum(0.5, 71, 30.0)[0] - np.exp(30j)) < 1e-12
    assert abs(C.gaussian_sum(0.5, 71, 0.0)[0] - 1.0) < 1e-12
    assert abs(C.gaussian_sum(0.5, 30, 30.0)[0] - np.exp(30j)) > 1e-2


def test_appendix_b_constants():
    """sum_{k>=1} e^{-4 pi^2 k} = 1/(1-e^{-4 pi^2}) - 1 ~ 7.15e-18, and
    PAPER.md:940-942: c = 2 sqrt(-log(sqrt(4 pi) tol)) ~ 12 at tol = 1e-16, m0 = c - 1 ~ 11."""
    q = math.exp(-4 * math.pi ** 2)
    s = q / (1.0 - q)          # = 1/(1-q) - 1 without cancellation
    assert abs(s - 7.15e-18) / 7.15e-18 < 0.01
    c = 2.0 * math.sqrt(-math.log(math.sqrt(4 * math.pi) * 1e-16))
    assert round(c) == 12
    assert C.m0_for_tol(1e-16, 0.5) == 11
    assert C.m0_for_tol(1e-12, 0.5) == 10
    assert C.m0_for_tol(1e-8, 0.5) == 8


@pytest.mark.parametrize("x", [30.0, 100.0])
@pytest.mark.parametrize("h", [0.2, 0.3, 0.5])
def test_scalar_rexii_fig1_threshold(x, h):
    """Fig. 1: the error drops to ~machine precision at
    M = ceil(x/h) + 11 and is large a few M below. Pins eq:bm, the windowed c_1/c_2
    sums and eq:modifiedRexi: a dropped or shifted term fails here."""
    M = C.M_rule(x, h)
    t = C.rexii_terms(h, M)
    err = abs(C.rexii_scalar(x, h, M, t)[0] - np.exp(1j * x))
    err_neg = abs(C.rexii_scalar(-x, h, M, t)[0] - np.exp(-1j * x))
    assert err < 1e-13 and err_neg < 1e-13
    err_lo = abs(C.rexii_scalar(x, h, M - 7)[0] - np.exp(1j * x))
    assert err_lo > 1e-5


def test_scalar_rexii_h1_floor_G8():
    """Reading G8: at h = 1 the plateau is the aliasing term e^{-4 pi (pi - h)} ~ 2.05e-12."""
    h, x = 1.0, 30.0
    M = C.M_rule(x, h) + 5
    err = abs(C.rexii_scalar(x, h, M)[0] - np.exp(1j * x))
    floor = math.exp(-4 * math.pi * (math.pi - h))
    assert 0.5 * floor < err < 2.0 * floor


def test_scalar_rexii_machine_precision_over_x():
    """at the minimal admissible M the error is close to machine precision for all x."""
    h, xmax = 0.5, 50.0
    M = C.M_rule(xmax, h)
    x = np.linspace(-xmax, xmax, 1001)
    err = np.abs(C.rexii_scalar(x, h, M) - np.exp(1j * x)).max()
    assert err < 1e-13


def test_rexi_and_rexii_scalar_equivalent():
    """in the scalar case the two single-sum forms are equivalent for real x."""
    h, M = 0.5, 80
    x = np.linspace(-30, 30, 301)
    d = np.abs(C.rexi_scalar(x, h, M) - C.rexii_scalar(x, h, M)).max()
    assert d < 1e-14


def test_remark3_coefficient_symmetries():
    """conj(c_{1,n}) = c_{1,-n}, conj(c_{2,n}) = -c_{2,-n}, alpha_n = conj(alpha_{-n})."""
    t = C.rexii_terms(0.5, 60)
    scale = np.abs(t.c1).max()
    assert np.abs(np.conj(t.c1) - t.c1[::-1]).max() < 1e-15 * scale
    assert np.abs(np.conj(t.c2) + t.c2[::-1]).max() < 1e-15 * np.abs(t.c2).max()
    assert np.abs(t.alpha - np.conj(t.alpha[::-1])).max() == 0.0
    assert t.N == 60 + 24 and len(t.n) == 2 * t.N + 1


def test_coefficients_extended_precision():
    """The longdouble table agrees with a 30-digit evaluation (reading G12)."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 30
    h, M = 0.1, 2000
    t = C.rexii_terms(h, M)
    mu, a, _ = C.appendix_a()
    hm = mpmath.mpf(h)
    for n in [0, 1, 17, 1000, M + 10, M + 24]:
        s1 = mpmath.mpc(0)
        for k in range(max(-24, n - M), min(24, n + M) + 1):
            re, im = C.A_APPENDIX_A[abs(k)]
            b = mpmath.exp(hm * hm) * mpmath.exp(mpmath.mpc(0, -1) * (n - k) * hm)
            s1 += mpmath.mpf(re) * b
        s1 *= hm
        j = n + t.N
        assert abs(complex(s1) - t.c1[j]) <= 1e-15 * max(1.0, abs(complex(s1)))


@pytest.mark.parametrize("D,tau,h,M", [
    (6, 1, 1.0, 38), (6, 1, 0.5, 65), (6, 1, 0.1, 278),          # Table 2
    (128, 1, 1.0, 580), (128, 1, 0.5, 1149), (128, 1, 0.1, 5698),  # Table 6
    (6, 50, 1.0, 1344), (6, 50, 0.5, 2677),                       # Table 3
])
def test_M_rule_reproduces_printed_M(D, tau, h, M):
    """eq:matrixAccuracyBound with rho = sqrt(2) pi D (reading G5)."""
    assert C.M_rule(tau * C.rho_lrsw(D), h, 11) == M


def test_M_rule_configs():
    """SURVEY.md 8(d) configs with m0(tol) of reading G9."""
    assert C.M_lrsw(512, 1.0, 0.5, 1e-8) == 4558
    assert C.M_lrsw(64, 0.02, 0.5, 1e-12) == 22
    assert C.M_lrsw(4096, 1.0, 0.5, 1e-12) == 36407


def test_rexi_beta_conjugate_symmetry_R2():
    """Reading R2: with the conjugate-symmetric Appendix A table,
    beta^Re_{-n} = conj(beta^Re_n); for a REAL matrix A and real f0 the term -n of
    eq:originalREXImatrix is then the complex conjugate of term n, so the real part of the full
    sum n = -N..N equals the half sum n = 0..N with Gamma_n. Checked on a random real 6x6."""
    h, M = 0.2, 150
    t = C.rexi_terms(h, M)
    assert np.abs(t.beta_re - np.conj(t.beta_re[::-1])).max() < 1e-15 * np.abs(t.beta_re).max()
    g = np.random.Generator(np.random.PCG64(3))
    B = g.standard_normal((6, 6))
    A = (B - B.T) * 2.0                       # real skew-symmetric, spectrum on iR
    f = g.standard_normal(6)
    I = np.eye(6)
    full = sum(np.real(b * np.linalg.solve(A + a * I, f)) for b, a in zip(t.beta_re, t.alpha))
    sel = t.n >= 0
    gam = np.where(t.n[sel] == 0, 1.0, 2.0)
    half = sum(gg * np.real(b * np.linalg.solve(A + a * I, f))
               for gg, b, a in zip(gam, t.beta_re[sel], t.alpha[sel]))
    assert np.abs(full - half).max() < 1e-12 * np.abs(full).max()


@pytest.mark.parametrize("tol", [1e-4, 1e-6, 1e-8, 1e-10, 1e-12])
def test_h_for_tol_meets_tol_scalar(tol):
    """NEXT-2 h optimiser (readings G8, G9): with h = h_for_tol(tol) and M from the rule, the
    scalar REXII meets tol over the whole admissible range (and uses ~h/0.5 x fewer terms)."""
    h = C.h_for_tol(tol)
    xmax = 60.0
    M = C.M_rule(xmax, h, C.m0_for_tol(tol, h))
    x = np.linspace(-xmax, xmax, 1201)
    err = np.abs(C.rexii_scalar(x, h, M) - np.exp(1j * x)).max()
    assert err < tol
    if tol >= 1e-8:
        assert h > 1.4 and M < 0.5 * C.M_rule(xmax, 0.5, C.m0_for_tol(tol, 0.5))


def test_oracle_refit_procedure_G18():
    """NEXT-2: the paper's l2 fit on Leja points (reading G18), done in fp64 (numpy lstsq; the
    system is ill-conditioned, so fp64 costs ~1 digit against the extended-precision planner fit,
    which meets the paper's "< 8e-15", test_capi_host.py): small defect on the core, small tail,
    and its REXII reproduces e^{ix} at the Fig. 1 threshold."""
    mu = float(C.MU_APPENDIX_A)
    a = C.fit_rational_gaussian(24, mu)
    x = np.linspace(-30, 30, 20001)
    assert np.abs(C.R_complex_form(x, mu, a) - C.psi(1.0, x)).max() < 1e-13
    xt = np.linspace(30, 1000, 20001)
    assert np.abs(C.R_complex_form(xt, mu, a)).max() < 5e-14
    assert a[24].imag == 0.0
    _, a0, _ = C.appendix_a()
    assert np.abs(a - a0).max() < 1e-2      # same mu and L: close to the printed table
    h, X = 0.5, 30.0
    M = C.M_rule(X, h)
    t = C.rexii_terms(h, M, mu=mu, a=a)
    assert abs(C.rexii_scalar(X, h, M, t)[0] - np.exp(1j * X)) < 3e-13
    # fitting only the core [0, 30] leaves a tail that ruins the REXI sum (why xmax = 100)
    b = C.fit_rational_gaussian(24, mu, K=100, xmax=30.0)
    tb = C.rexii_terms(h, M, mu=mu, a=b)
    assert abs(C.rexii_scalar(X, h, M, tb)[0] - np.exp(1j * X)) > 1e-11
