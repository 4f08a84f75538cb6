"""NEXT-3 oracle pins: the Sec. 3.2 test matrices (Fig. 2) with the matrix
forms of REXII, REXI and REXIE evaluated by dense solves, against scipy's Pade expm."""
import numpy as np
import pytest

from oracle import coeffs as C
from oracle import matrix as X


def test_test_matrices_spectra():
    A1, x1 = X.advection_A1()
    assert np.abs(A1 + A1.T).max() == 0.0                 # skew-symmetric
    ev = np.linalg.eigvals(A1)
    assert np.abs(ev.real).max() < 1e-10 and np.abs(ev.imag).max() <= 70.0 + 1e-9
    A2, x2 = X.schrodinger_A2()
    ev2 = np.linalg.eigvals(A2)                            # i[-4900, 0]
    assert np.abs(ev2.real).max() < 1e-9
    assert ev2.imag.min() > -4900.0 - 1e-6 and ev2.imag.max() < 1e-9
    assert np.abs(A2 + A2.conj().T).max() < 1e-9           # skew-Hermitian


def test_fig2a_rexii_threshold_A1():
    """Fig. 2(a): REXII on A_1 follows tau rho(A) <= (M - 11) h (eq:matrixAccuracyBound)."""
    A1, x = X.advection_A1()
    f = X.f0(x)
    ex = X.expm_apply(A1, f, 1.0)
    for h in (0.5, 0.2):
        M = C.M_rule(70.0, h)
        assert X.rel_l2(X.rexii_matrix(A1, f, 1.0, h, M), ex) < 1e-13
        assert X.rel_l2(X.rexii_matrix(A1, f, 1.0, h, M - int(15 / h)), ex) > 1e-9
    # Remark 3: half sum + Re == full sum for real A, f
    M = C.M_rule(70.0, 0.5)
    full = X.rexii_matrix(A1, f, 1.0, 0.5, M, half=False)
    assert np.abs(full.imag).max() < 1e-12
    assert X.rel_l2(full.real, X.rexii_matrix(A1, f, 1.0, 0.5, M)) < 1e-13


def test_fig2b_rexi_stagnates_A1():
    """Fig. 2(b): the original REXI does not follow the bound; at the REXII M it stays far
    from the exponential."""
    A1, x = X.advection_A1()
    f = X.f0(x)
    ex = X.expm_apply(A1, f, 1.0)
    for h in (0.5, 0.2):
        M = C.M_rule(70.0, h) + 10
        assert X.rel_l2(X.rexi_matrix(A1, f, 1.0, h, M), ex) > 1e-7


def test_fig2c_rexie_shift_A2():
    """Fig. 2(c): REXIE with the shift nu = -2450 i (Remark 1) on A_2 converges at
    tau rho(A') <= (M - 11) h with rho(A') = 2450; without the shift the same M fails."""
    A2, x = X.schrodinger_A2()
    f = X.f0(x)
    ex = X.expm_apply(A2, f, 1.0)
    M = C.M_rule(2450.0, 0.5)
    assert X.rel_l2(X.rexie_matrix(A2, f, 1.0, 0.5, M, nu=-2450j), ex) < 1e-11
    assert X.rel_l2(X.rexie_matrix(A2, f, 1.0, 0.5, M - 50, nu=-2450j), ex) > 1e-3
    # without the shift the same M covers only |lambda| <= (M - 11) h = 2450 of the spectrum
    # i[-4900, 0] (eq:matrixAccuracyBound): beyond it R(x) ~ 0, so the error is the part of f0
    # on the eigenvectors with |lambda| > 2450 (A_2 is normal: e^{A_2} is unitary)
    H = (A2 / 1j).real                      # A_2 = i H, H real symmetric
    w, V = np.linalg.eigh(H)
    c = V.T @ f
    tail = np.linalg.norm(c[np.abs(w) > 2450.0]) / np.linalg.norm(c)
    err0 = X.rel_l2(X.rexie_matrix(A2, f, 1.0, 0.5, M, nu=0.0), ex)
    assert tail > 1e-6 and abs(err0 - tail) < 1e-3 * tail, (err0, tail)
