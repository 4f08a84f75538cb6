"""NEXT-3 generic matrices — ORACLE (test infrastructure only; see oracle/coeffs.py header).

The test matrices of Sec. 3.2 and the matrix forms of REXII, REXI and REXIE
evaluated literally with dense shifted solves (numpy.linalg.solve), for Fig. 2.

Reading G19: A_1 has n = 70 periodic unknowns x_j = j/70 on [0, 1) ("discretization
step 1/70"), A_1 f = (f_{j+1} - f_{j-1}) / (2 dx): skew-symmetric, eigenvalues in i[-70, 70].
A_2 has n = 70 periodic unknowns x_j = -1 + j/35 on [-1, 1) (step 1/35),
A_2 f = i (f_{j+1} - 2 f_j + f_{j-1}) / dx^2: eigenvalues in i[-4900, 0], shift nu = -2450 i.
f_0 = (2 + cos(2 pi x))^{-1} on the grid.
"""
from __future__ import annotations

import numpy as np

from . import coeffs as C


def circulant(first_col):
    n = len(first_col)
    return np.array([[first_col[(i - j) % n] for j in range(n)] for i in range(n)])


def advection_A1(n=70):
    """Second-order centred FD of d/dx, periodic, dx = 1/n."""
    dx = 1.0 / n
    c = np.zeros(n)
    c[1] = -1.0 / (2 * dx)     # row i: (f_{i+1} - f_{i-1}) / (2 dx)  -> A[i, i+1] = +, A[i, i-1] = -
    c[n - 1] = 1.0 / (2 * dx)
    A = circulant(c)
    x = np.arange(n) * dx
    return A, x


def schrodinger_A2(n=70):
    """Second-order FD of i d^2/dx^2, periodic on [-1, 1), dx = 2/n = 1/35."""
    dx = 2.0 / n
    c = np.zeros(n, dtype=np.complex128)
    c[0] = -2j / dx ** 2
    c[1] = 1j / dx ** 2
    c[n - 1] = 1j / dx ** 2
    A = circulant(c)
    x = -1.0 + np.arange(n) * dx
    return A, x


def f0(x):
    """(2 + cos(2 pi x))^{-1}."""
    return 1.0 / (2.0 + np.cos(2.0 * np.pi * x))


def rexii_matrix(A, f, tau, h, M, half=True):
    """eq:REXI_Modified_matrix applied to f with dense solves; half=True uses
    Remark 3's half sum + Re (real A, f; eq:modifiedRexiMatrixReducedSum)."""
    t = C.rexii_terms(h, M)
    n = A.shape[0]
    I = np.eye(n)
    acc = np.zeros(n, dtype=np.complex128)
    sel = (t.n >= 0) if half else np.ones_like(t.n, dtype=bool)
    for nn, al, C1, C2 in zip(t.n[sel], t.alpha[sel], t.C1[sel], t.C2[sel]):
        gam = (1.0 if nn == 0 else 2.0) if half else 1.0
        g1 = np.linalg.solve(al * I + tau * A, f)
        g2 = np.linalg.solve(np.conj(al) * I - tau * A, g1)
        acc += gam * (C2 * g1 + (C1 - C2 * np.conj(al)) * g2)
    return acc.real if half else acc


def rexi_matrix(A, f, tau, h, M):
    """eq:originalREXImatrix: sum_{n=-N}^{N} Re(beta^Re_n (tau A + alpha_n I)^{-1}) f."""
    t = C.rexi_terms(h, M)
    n = A.shape[0]
    I = np.eye(n)
    acc = np.zeros(n, dtype=np.complex128)
    for al, bR in zip(t.alpha, t.beta_re):
        acc += bR * np.linalg.solve(tau * A + al * I, f)
    return acc.real


def rexie_matrix(A, f, tau, h, M, nu=0.0):
    """eq:REXIE with Remark 1's shift:
    e^{tau A} f ~ e^{tau nu} sum_n [Re(beta^Re_n (tau A' + alpha_n)^{-1} f) + i Re(beta^Im_n (...)^{-1} f)],
    A' = A - nu I (A' = iB' with B' real, f real)."""
    t = C.rexi_terms(h, M)
    n = A.shape[0]
    I = np.eye(n)
    Ap = A - nu * I
    re = np.zeros(n)
    im = np.zeros(n)
    for al, bR, bI in zip(t.alpha, t.beta_re, t.beta_im):
        g = np.linalg.solve(tau * Ap + al * I, f)
        re += np.real(bR * g)
        im += np.real(bI * g)
    return np.exp(tau * nu) * (re + 1j * im)


def expm_apply(A, f, tau):
    import scipy.linalg
    return scipy.linalg.expm(tau * A) @ f


def rel_l2(a, b):
    """The error of PAPER.md:390-392: ||a - b||_2 / ||b||_2."""
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
