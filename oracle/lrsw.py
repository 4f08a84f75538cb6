"""LRSW REXII step — ORACLE (test infrastructure only; see oracle/coeffs.py header).

Python driver around ``rexi_oracle.c`` (naive DFT + dense per-mode 3x3 solves),
plus the exact per-mode propagator and a brute-force matrix exponential used to
pin it. Follows PAPER.md Sec. 4 step by step.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

from . import coeffs

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rexi_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "librexi_oracle.so")
_lib = None
_lock = threading.Lock()

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build(force=False):
    """Compile the C oracle with gcc (-O2, OpenMP). Building the checker is not using it."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                           "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            L.oracle_num_threads.argtypes = [ctypes.c_int]
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_dft2_forward.argtypes = [ctypes.c_int, _dp, _dp]
            L.oracle_dft2_inverse_real.argtypes = [ctypes.c_int, _dp, _dp]
            L.oracle_rexii_pole_sum.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                                _dp, _dp, _dp, _dp, ctypes.c_long, _ip, _ip, _dp, _dp]
            L.oracle_rexi_pole_sum.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                               _dp, _dp, ctypes.c_long, _ip, _ip, _dp, _dp]
            _lib = L
    return _lib


def num_threads(n=0):
    """Set (n > 0) and return the OpenMP thread count the oracle uses."""
    return lib().oracle_num_threads(int(n))


def _d(a):
    return a.ctypes.data_as(_dp)


def _cri(z):
    """complex128 array -> contiguous interleaved float64 view."""
    z = np.ascontiguousarray(z, dtype=np.complex128)
    return z.view(np.float64)


# ---------------------------------------------------------------------------
# Transforms (S1 / S5): "all computations ... in Fourier space"
# ---------------------------------------------------------------------------
def dft2(X):
    """Xhat[l, k] = D^-2 sum_{y,x} X[y, x] exp(-2 pi i (k x + l y)/D)  (naive, O(D^3))."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    D = X.shape[0]
    out = np.empty((D, D), dtype=np.complex128)
    lib().oracle_dft2_forward(D, _d(X), _d(out.view(np.float64)))
    return out


def idft2_real(Xhat):
    """X[y, x] = Re sum_{l,k} Xhat[l, k] exp(+2 pi i (k x + l y)/D)  (naive, O(D^3))."""
    Xhat = np.ascontiguousarray(Xhat, dtype=np.complex128)
    D = Xhat.shape[0]
    out = np.empty((D, D), dtype=np.float64)
    lib().oracle_dft2_inverse_real(D, _d(Xhat.view(np.float64)), _d(out))
    return out


def wavenumbers(D):
    """k for index j = 0..D-1: j (j < D/2) else j - D."""
    j = np.arange(D)
    return np.where(j < D // 2, j, j - D)


def symbols(D, tau, nyquist_zero=True):
    """tau-scaled first-derivative symbols 2 pi k tau per index (G3), Nyquist zeroed (G2)."""
    K = 2.0 * math.pi * wavenumbers(D).astype(np.float64) * tau
    if nyquist_zero:
        K[D // 2] = 0.0
    return K


# ---------------------------------------------------------------------------
# Pole sums (S2 + S3): dense per-mode solves, ascending n
# ---------------------------------------------------------------------------
def rexii_pole_sum(D, tau, fhat_modes, mode_l, mode_k, alpha, C1, C2, gamma, nyquist_zero=True):
    """acc[m, c] = sum_{n} Gamma_n (C2_n g1 + (C1_n - C2_n alpha_{-n}) g2) for each listed mode.

    fhat_modes: (n_modes, 3) complex (eta, u, v) Fourier coefficients."""
    f = np.ascontiguousarray(fhat_modes, dtype=np.complex128).reshape(-1, 3)
    nm = f.shape[0]
    acc = np.zeros((nm, 3), dtype=np.complex128)
    ml = np.ascontiguousarray(mode_l, dtype=np.int32)
    mk = np.ascontiguousarray(mode_k, dtype=np.int32)
    a, c1, c2 = _cri(alpha), _cri(C1), _cri(C2)
    g = np.ascontiguousarray(gamma, dtype=np.float64)
    lib().oracle_rexii_pole_sum(int(D), float(tau), int(bool(nyquist_zero)), int(len(g)),
                                _d(a), _d(c1), _d(c2), _d(g), nm,
                                ml.ctypes.data_as(_ip), mk.ctypes.data_as(_ip),
                                _d(f.view(np.float64)), _d(acc.view(np.float64)))
    return acc


def _solve3_ld(A, r):
    """x = A^-1 r for a batch of 3x3 complex longdouble systems (A: (m, 3, 3), r: (m, 3)) by
    Cramer's rule: x_i = det(A with column i replaced by r) / det(A)."""
    def det(M):
        return (M[:, 0, 0] * (M[:, 1, 1] * M[:, 2, 2] - M[:, 1, 2] * M[:, 2, 1])
                - M[:, 0, 1] * (M[:, 1, 0] * M[:, 2, 2] - M[:, 1, 2] * M[:, 2, 0])
                + M[:, 0, 2] * (M[:, 1, 0] * M[:, 2, 1] - M[:, 1, 1] * M[:, 2, 0]))
    d = det(A)
    x = np.empty_like(r)
    for i in range(3):
        Ai = A.copy()
        Ai[:, :, i] = r
        x[:, i] = det(Ai) / d
    return x


def rexii_pole_sum_ld(D, tau, fhat_modes, mode_l, mode_k, terms_ld, begin=0, end=None):
    """Extended-precision reference of rexii_pole_sum for poles [begin, end) of the half-sum
    (test infrastructure: the "long-double truth" of DESIGN.md reading R1). Every quantity is
    complex longdouble (x87, 64-bit mantissa: 2^11 x the fp64 precision): the unrounded
    coefficient table (coeffs.rexii_half_terms_ld), the tau-scaled symbols 2 pi k tau (G3,
    Nyquist zeroed, G2) with pi in longdouble, and per mode and pole the two shifted systems of
    PAPER.md:429-431 solved by Cramer's rule (not the fp64 oracle's pivoted elimination),
    accumulated in ascending n as in the display PAPER.md:432-434:
        acc += Gamma_n [C2_n g1 + (C1_n - C2_n conj(alpha_n)) g2],
        (alpha_n I + tau A) g1 = f0,  (conj(alpha_n) I - tau A) g2 = g1.
    fhat_modes: (n_modes, 3) complex; returns (n_modes, 3) clongdouble."""
    CL, LDt = np.clongdouble, np.longdouble
    n, alpha, C1, C2, gamma = terms_ld
    end = len(n) if end is None else end
    pi = LDt(4) * np.arctan(LDt(1))
    kk = wavenumbers(D).astype(LDt)
    sym = LDt(2) * pi * kk * LDt(tau)
    sym[D // 2] = LDt(0)
    kx = sym[np.asarray(mode_k)].astype(CL)
    ky = sym[np.asarray(mode_l)].astype(CL)
    nm = len(kx)
    t = CL(LDt(tau))
    # tau A-hat per mode: [[0, -i kx, -i ky], [-i kx, 0, tau], [-i ky, -tau, 0]]
    B = np.zeros((nm, 3, 3), dtype=CL)
    B[:, 0, 1] = -1j * kx
    B[:, 0, 2] = -1j * ky
    B[:, 1, 0] = -1j * kx
    B[:, 2, 0] = -1j * ky
    B[:, 1, 2] = t
    B[:, 2, 1] = -t
    eye = np.eye(3, dtype=CL)[None]
    f0 = np.asarray(fhat_modes).astype(CL).reshape(-1, 3)
    acc = np.zeros((nm, 3), dtype=CL)
    for j in range(begin, end):
        a = alpha[j]
        ab = np.conj(a)
        g1 = _solve3_ld(a * eye + B, f0)
        g2 = _solve3_ld(ab * eye - B, g1)
        acc += gamma[j] * (C2[j] * g1 + (C1[j] - C2[j] * ab) * g2)
    return acc


def rexi_pole_sum(D, tau, fhat_modes, mode_l, mode_k, alpha, beta, nyquist_zero=True):
    f = np.ascontiguousarray(fhat_modes, dtype=np.complex128).reshape(-1, 3)
    nm = f.shape[0]
    acc = np.zeros((nm, 3), dtype=np.complex128)
    ml = np.ascontiguousarray(mode_l, dtype=np.int32)
    mk = np.ascontiguousarray(mode_k, dtype=np.int32)
    a, b = _cri(alpha), _cri(beta)
    lib().oracle_rexi_pole_sum(int(D), float(tau), int(bool(nyquist_zero)), int(len(alpha)),
                               _d(a), _d(b), nm, ml.ctypes.data_as(_ip), mk.ctypes.data_as(_ip),
                               _d(f.view(np.float64)), _d(acc.view(np.float64)))
    return acc


def all_modes(D):
    l, k = np.meshgrid(np.arange(D), np.arange(D), indexing="ij")
    return l.ravel().astype(np.int32), k.ravel().astype(np.int32)


def spectral_fields(eta, u, v):
    """(D, D, 3) complex Fourier coefficients of the three real fields."""
    return np.stack([dft2(eta), dft2(u), dft2(v)], axis=-1)


def rexii_step(eta, u, v, tau, h, M, nyquist_zero=True, terms=None, modes=None):
    """One REXII step e^{tau A} f0 on the D x D grid.

    1. naive DFT of (eta, u, v)                      (Alg. 1 line 1)
    2. for n = 0..N: two dense per-mode solves, acc += g3
    3. Re(inverse DFT(acc))
    If ``modes`` = (l, k) is given, only those modes are processed; all others are
    taken as zero (exact when the input spectrum vanishes there)."""
    D = eta.shape[0]
    n, alpha, C1, C2, gamma = (terms or coeffs.rexii_terms(h, M)).half()
    F = spectral_fields(eta, u, v)
    if modes is None:
        ml, mk = all_modes(D)
    else:
        ml, mk = modes
    acc = rexii_pole_sum(D, tau, F[ml, mk, :], ml, mk, alpha, C1, C2, gamma, nyquist_zero)
    A = np.zeros((D, D, 3), dtype=np.complex128)
    A[ml, mk, :] = acc
    return tuple(idft2_real(A[..., c]) for c in range(3))


def rexi_step(eta, u, v, tau, h, M, nyquist_zero=True, modes=None):
    """Original REXI step, eq:originalREXImatrix, full sum n = -N..N."""
    D = eta.shape[0]
    t = coeffs.rexi_terms(h, M)
    F = spectral_fields(eta, u, v)
    ml, mk = all_modes(D) if modes is None else modes
    acc = rexi_pole_sum(D, tau, F[ml, mk, :], ml, mk, t.alpha, t.beta_re, nyquist_zero)
    A = np.zeros((D, D, 3), dtype=np.complex128)
    A[ml, mk, :] = acc
    return tuple(idft2_real(A[..., c]) for c in range(3))


# ---------------------------------------------------------------------------
# Exact reference (reading G15): the per-mode propagator e^{tau Ahat}
# ---------------------------------------------------------------------------
def exact_propagator_modes(Kx, Ky, tau):
    """e^{B}, B = tau*Ahat (skew-Hermitian, eigenvalues {0, +-i w}, w^2 = Kx^2 + Ky^2 + tau^2):
    e^B = I + (sin w / w) B + ((1 - cos w)/w^2) B^2  (closed-form eigen-decomposition).
    Kx, Ky already tau-scaled. Returns (..., 3, 3) complex."""
    Kx = np.asarray(Kx, dtype=np.float64)
    Ky = np.asarray(Ky, dtype=np.float64)
    shp = np.broadcast(Kx, Ky).shape
    B = np.zeros(shp + (3, 3), dtype=np.complex128)
    B[..., 0, 1] = -1j * Kx
    B[..., 0, 2] = -1j * Ky
    B[..., 1, 0] = -1j * Kx
    B[..., 2, 0] = -1j * Ky
    B[..., 1, 2] = tau
    B[..., 2, 1] = -tau
    w = np.sqrt(Kx * Kx + Ky * Ky + tau * tau)
    with np.errstate(invalid="ignore", divide="ignore"):
        s1 = np.where(w > 0, np.sin(w) / np.where(w > 0, w, 1.0), 1.0)
        s2 = np.where(w > 1e-4, (1.0 - np.cos(w)) / np.where(w > 0, w * w, 1.0),
                      0.5 - w * w / 24.0)
    B2 = B @ B
    E = np.eye(3, dtype=np.complex128) + s1[..., None, None] * B + s2[..., None, None] * B2
    return E


def exact_spectral(F, tau, nyquist_zero=True):
    """Apply e^{tau Ahat} per mode to F (D, D, 3) complex."""
    D = F.shape[0]
    K = symbols(D, tau, nyquist_zero)
    Ky, Kx = np.meshgrid(K, K, indexing="ij")   # row l -> Ky, column k -> Kx
    E = exact_propagator_modes(Kx, Ky, tau)
    return np.einsum("lkij,lkj->lki", E, F)


def exact_step(eta, u, v, tau, nyquist_zero=True):
    F = spectral_fields(eta, u, v)
    G = exact_spectral(F, tau, nyquist_zero)
    return tuple(idft2_real(G[..., c]) for c in range(3))


# ---------------------------------------------------------------------------
# Brute force (tiny grids): the full 3D^2 x 3D^2 real operator and Pade expm
# ---------------------------------------------------------------------------
def lrsw_operator_dense(D, nyquist_zero=True):
    """The real matrix A of PAPER.md:419-426 on the D x D grid with spectral first
    derivatives (symbol 2 pi i k, Nyquist zeroed), unknowns ordered (eta, u, v) each
    row-major [y][x]. Built from DFT matrices: d/dx = F^-1 diag(i 2 pi k) F."""
    j = np.arange(D)
    F1 = np.exp(-2j * np.pi * np.outer(j, j) / D) / D           # forward, scaled
    Fi = np.exp(2j * np.pi * np.outer(j, j) / D)                # inverse
    k = 2.0 * np.pi * wavenumbers(D).astype(np.float64)
    if nyquist_zero:
        k[D // 2] = 0.0
    d1 = (Fi @ np.diag(1j * k) @ F1).real                      # 1-D derivative (real)
    I1 = np.eye(D)
    Dx = np.kron(I1, d1)      # acts along x (fastest index)
    Dy = np.kron(d1, I1)      # acts along y
    n = D * D
    Z = np.zeros((n, n))
    Id = np.eye(n)
    A = np.block([[Z, -Dx, -Dy], [-Dx, Z, Id], [-Dy, -Id, Z]])
    return A


def brute_force_step(eta, u, v, tau, nyquist_zero=True):
    import scipy.linalg
    D = eta.shape[0]
    A = lrsw_operator_dense(D, nyquist_zero)
    f = np.concatenate([eta.ravel(), u.ravel(), v.ravel()])
    g = scipy.linalg.expm(tau * A) @ f
    n = D * D
    return g[:n].reshape(D, D), g[n:2 * n].reshape(D, D), g[2 * n:].reshape(D, D)
