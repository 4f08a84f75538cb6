"""REXI / REXII coefficient generation — ORACLE (test infrastructure only).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product path
(``paper_2008_11607_b200``) never does, and this package never imports the
product path.

Everything here follows arXiv:2008.11607 (``/root/reference/PAPER.md``) step by
step, in the paper's order and notation. Coefficients are generated in x87
extended precision (numpy.longdouble, 64-bit mantissa) and rounded to fp64 at
the end, so the oracle's own rounding stays below the fp64 product's.

Citations are ``PAPER.md:<line>`` plus the LaTeX label.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

LD = np.longdouble

# ---------------------------------------------------------------------------
# Appendix A, PAPER.md:815-851 (tab:coef_al). L = 24, mu, a_0..a_24.
# Reading G1: the printed sign column applies to the real part only.
# (Typed independently of the product planner's copy; tests compare both with
#  tests/golden/appendix_a.txt.)
# ---------------------------------------------------------------------------
MU_APPENDIX_A = "-5.133333333333333"
A_APPENDIX_A = [  # (Re a_l, Im a_l) as printed, l = 0..24
    ("-6.520430828919864e+01", "0.0"),
    ("4.261818064131437e+01", "2.761406741120911e+01"),
    ("-9.801650304425239e+00", "-2.189295463610722e+01"),
    ("-1.054225194693395e+00", "6.791786454153551e+00"),
    ("7.950505668209775e-01", "-8.904997258367445e-01"),
    ("-1.218558380859130e-01", "3.321241563407446e-02"),
    ("7.365401806949337e-03", "2.212802103193251e-03"),
    ("-2.801087265991056e-04", "-5.566945197754387e-04"),
    ("1.254835436432561e-04", "-2.467200513365371e-04"),
    ("2.295472292491263e-04", "-8.494118951459107e-05"),
    ("1.858484460459430e-04", "9.242889460185034e-05"),
    ("4.068056518449676e-05", "1.653479957565515e-04"),
    ("-8.341508001647741e-05", "1.045331460447588e-04"),
    ("-9.970528169841103e-05", "-5.856228484297677e-06"),
    ("-3.499639858693093e-05", "-6.129059473910835e-05"),
    ("2.295021920298455e-05", "-4.099832469456381e-05"),
    ("2.931048772724314e-05", "1.708815129697846e-07"),
    ("7.502088478301169e-06", "1.525082051744077e-05"),
    ("-5.815291167450100e-06", "6.919604247338349e-06"),
    ("-4.069948458364005e-06", "-1.440010113050771e-06"),
    ("7.932524475429588e-08", "-1.794169428574330e-06"),
    ("6.120984882186265e-07", "-1.131894636585849e-07"),
    ("5.531365159161319e-08", "1.585749903175946e-07"),
    ("-2.867805871375946e-08", "1.239499740327838e-08"),
    ("-1.143081277095316e-09", "-2.763239274253499e-09"),
]
L_APPENDIX_A = 24  # PAPER.md:282 "where L=24"


def appendix_a(dtype=np.float64):
    """(mu, a) with a[l + L] = a_l for l = -L..L and a_{-l} = conj(a_l)
    (PAPER.md:851 caption "with a_l = conj(a_{-l})")."""
    L = L_APPENDIX_A
    mu = dtype(MU_APPENDIX_A) if dtype is not LD else LD(MU_APPENDIX_A)
    re = np.array([LD(r) for r, _ in A_APPENDIX_A], dtype=LD)
    im = np.array([LD(i) for _, i in A_APPENDIX_A], dtype=LD)
    a_re = np.concatenate([re[:0:-1], re])          # l = -L..L, Re a_{-l} = Re a_l
    a_im = np.concatenate([-im[:0:-1], im])         # Im a_{-l} = -Im a_l
    if dtype is LD:
        return mu, a_re, a_im
    return float(mu), (a_re.astype(np.float64) + 1j * a_im.astype(np.float64)), L


# ---------------------------------------------------------------------------
# Step 1 — Gaussian basis and b_m
# ---------------------------------------------------------------------------
def psi(h, x):
    """eq:psi: psi_h(x) = (4 pi)^(-1/2) exp(-x^2 / (4 h^2))."""
    x = np.asarray(x, dtype=np.float64)
    return np.exp(-x * x / (4.0 * h * h)) / math.sqrt(4.0 * math.pi)


def b_coeffs_ld(h, M):
    """eq:bm: b_m = e^{-imh} e^{h^2}, m = -M..M (longdouble re, im).

    The phase m*h is formed in extended precision (reading G12)."""
    if not (0.0 < h < math.pi):
        raise ValueError("h must lie in (0, pi) (PAPER.md:98)")
    m = np.arange(-M, M + 1, dtype=LD)
    hh = LD(h)
    ph = m * hh
    eh2 = np.exp(hh * hh)
    return eh2 * np.cos(ph), -eh2 * np.sin(ph)


def gaussian_sum(h, M, x):
    """eq:eixsumM: e^{ix} ~ sum_{m=-M}^{M} b_m psi_h(x + m h)."""
    bre, bim = b_coeffs_ld(h, M)
    b = bre.astype(np.float64) + 1j * bim.astype(np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    out = np.zeros(x.shape, dtype=np.complex128)
    for j, m in enumerate(range(-M, M + 1)):
        out += b[j] * psi(h, x + m * h)
    return out


# ---------------------------------------------------------------------------
# Step 2 — rational approximation of the Gaussian
# ---------------------------------------------------------------------------
def R_complex_form(x, mu=None, a=None):
    """eq:ratapproxgaush1: R(x) = Re sum_{l=-L}^{L} a_l/(ix + mu + il)."""
    if mu is None:
        mu, a, L = appendix_a()
    L = (len(a) - 1) // 2
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    s = np.zeros(x.shape, dtype=np.complex128)
    for j, l in enumerate(range(-L, L + 1)):
        s += a[j] / (1j * x + mu + 1j * l)
    return s.real


def R_real_form(x, mu=None, a=None):
    """eq:A(x,mu), PAPER.md:143-147 (symmetric real form, a_{-l} = conj(a_l))."""
    if mu is None:
        mu, a, L = appendix_a()
    L = (len(a) - 1) // 2
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    x2 = x * x
    out = a[L].real * mu / (x2 + mu * mu)
    for l in range(1, L + 1):
        al = a[L + l]
        num = 2.0 * mu * al.real * (mu * mu + l * l + x2) + 2.0 * l * al.imag * (mu * mu + l * l - x2)
        den = x2 * x2 + 2.0 * (mu * mu - l * l) * x2 + (mu * mu + l * l) ** 2
        out = out + num / den
    return out


def leja_points(K, xmax, ncand=30001):
    """Reading G18: the Leja sequence on [0, xmax] from x_1 = 0 ("the same strategy
    that is used for ... interpolation with Leja points"): x_{k+1} maximises prod_j |x - x_j|
    over a uniform candidate grid."""
    cand = np.linspace(0.0, xmax, ncand)
    pts = [0.0]
    logp = np.log(np.abs(cand) + 1e-300)
    used = np.zeros(ncand, dtype=bool)
    used[0] = True
    for _ in range(1, K):
        score = np.where(used, -np.inf, logp)
        i = int(np.argmax(score))
        used[i] = True
        pts.append(cand[i])
        logp = logp + np.log(np.abs(cand - cand[i]) + 1e-300)
    return np.array(pts)


def design_matrix(x, mu, L):
    """G(x, mu, L) of PAPER.md:155-162: columns for y = [a0, Re a_1..Re a_L, Im a_1..Im a_L]
    of the real form eq:A(x,mu)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    x2 = x * x
    cols = [mu / (x2 + mu * mu)]
    dens = [x2 * x2 + 2.0 * (mu * mu - l * l) * x2 + (mu * mu + l * l) ** 2 for l in range(1, L + 1)]
    for l in range(1, L + 1):
        cols.append(2.0 * mu * (mu * mu + l * l + x2) / dens[l - 1])
    for l in range(1, L + 1):
        cols.append(2.0 * l * (mu * mu + l * l - x2) / dens[l - 1])
    return np.stack(cols, axis=-1)


def fit_rational_gaussian(L=24, mu=-5.133333333333333, K=200, xmax=100.0):
    """NEXT-2: eq:minl2approx — least squares of psi_1 - R on K Leja points
    on [0, xmax] (reading G18; xmax = 100 so the tail of R, which the REXI sums evaluate, stays
    small). Returns a[0..2L] with a[L + l] = a_l, a_{-l} = conj(a_l)."""
    x = leja_points(K, xmax)
    y, *_ = np.linalg.lstsq(design_matrix(x, mu, L), psi(1.0, x), rcond=None)
    a = np.zeros(2 * L + 1, dtype=np.complex128)
    a[L] = y[0]
    for l in range(1, L + 1):
        a[L + l] = y[l] + 1j * y[L + l]
        a[L - l] = np.conj(a[L + l])
    return a


# ---------------------------------------------------------------------------
# Step 3 — single-sum coefficient tables
# ---------------------------------------------------------------------------
@dataclass
class RexiiTerms:
    """Term table of eq:modifiedRexi / eq:REXI_Modified_matrix for n = -N..N."""
    h: float
    M: int
    L: int
    N: int
    mu: float
    n: np.ndarray          # -N..N (int64)
    alpha: np.ndarray      # alpha_n = h(mu + i n)
    c1: np.ndarray         # c_{1,n}
    c2: np.ndarray         # c_{2,n}
    C1: np.ndarray         # C_{1,n} = c_{1,n} h mu + c_{2,n} h n
    C2: np.ndarray         # C_{2,n} = i c_{2,n}

    def half(self):
        """Remark 3 (eq:modifiedRexiMatrixReducedSum): n = 0..N
        with Gamma_0 = 1, Gamma_n = 2."""
        sel = self.n >= 0
        gamma = np.where(self.n[sel] == 0, 1.0, 2.0)
        return self.n[sel], self.alpha[sel], self.C1[sel], self.C2[sel], gamma


def _windowed(h, M, L, wk_re, wk_im, bre, bim, N):
    """h * sum_{k=L1(n)}^{L2(n)} w_k b_{n-k}, L1 = max(-L, n-M), L2 = min(L, n+M)
     for n = -N..N, with w_k = wk_re + i wk_im (longdouble).
    The sum over k is taken in ascending k for every n, as written."""
    n = np.arange(-N, N + 1)
    out_re = np.zeros(2 * N + 1, dtype=LD)
    out_im = np.zeros(2 * N + 1, dtype=LD)
    for k in range(-L, L + 1):
        m = n - k
        ok = (m >= -M) & (m <= M)          # k in [L1(n), L2(n)]  <=>  |n-k| <= M
        idx = (m + M)[ok]
        br, bi = bre[idx], bim[idx]
        wr, wi = wk_re[k + L], wk_im[k + L]
        out_re[ok] += wr * br - wi * bi
        out_im[ok] += wr * bi + wi * br
    hh = LD(h)
    return hh * out_re, hh * out_im


def _rexii_terms_ld(h, M, mu=None, a=None):
    """The REXII term table in extended precision: (L, N, mu_ld, n, c1r, c1i, c2r, c2i, C1r, C1i,
    C2r, C2i), every array longdouble (eq:modifiedRexi, eq:REXI_Modified_matrix), N = M + L."""
    if mu is None:
        mu_ld, a_re, a_im = appendix_a(LD)
        L = L_APPENDIX_A
    else:
        a = np.asarray(a, dtype=np.complex128)
        L = (len(a) - 1) // 2
        mu_ld = LD(mu)
        a_re = a.real.astype(LD)
        a_im = a.imag.astype(LD)
    N = M + L
    bre, bim = b_coeffs_ld(h, M)
    zero = np.zeros_like(a_re)
    # c_{1,n} = h sum Re(a_k) b_{n-k};  c_{2,n} = h sum Im(a_k) b_{n-k}
    c1r, c1i = _windowed(h, M, L, a_re, zero, bre, bim, N)
    c2r, c2i = _windowed(h, M, L, a_im, zero, bre, bim, N)
    n = np.arange(-N, N + 1)
    hh = LD(h)
    n_ld = n.astype(LD)
    # C_{1,n} = c_{1,n} h mu + c_{2,n} h n ;  C_{2,n} = i c_{2,n}
    C1r = c1r * hh * mu_ld + c2r * hh * n_ld
    C1i = c1i * hh * mu_ld + c2i * hh * n_ld
    C2r, C2i = -c2i, c2r
    return L, N, mu_ld, n, c1r, c1i, c2r, c2i, C1r, C1i, C2r, C2i


def rexii_terms(h, M, mu=None, a=None):
    """The REXII term table (eq:modifiedRexi, eq:REXI_Modified_matrix), N = M + L, rounded once
    to fp64. Default table: Appendix A; or (mu, a[0..2L]) with a[L + l] = a_l (e.g. a NEXT-2
    refit)."""
    L, N, mu_ld, n, c1r, c1i, c2r, c2i, C1r, C1i, C2r, C2i = _rexii_terms_ld(h, M, mu, a)
    hh = LD(h)
    n_ld = n.astype(LD)
    f = lambda r, i: r.astype(np.float64) + 1j * i.astype(np.float64)
    alpha = (float(hh * mu_ld) + 1j * (hh * n_ld).astype(np.float64))
    return RexiiTerms(h=h, M=M, L=L, N=N, mu=float(mu_ld), n=n, alpha=alpha,
                      c1=f(c1r, c1i), c2=f(c2r, c2i), C1=f(C1r, C1i), C2=f(C2r, C2i))


def rexii_half_terms_ld(h, M):
    """Remark 3's half-sum table n = 0..N NOT rounded to fp64: complex
    longdouble (clongdouble) alpha_n, C_{1,n}, C_{2,n} and Gamma_n — the coefficients of the
    extended-precision reference lrsw.rexii_pole_sum_ld (test infrastructure, R1)."""
    L, N, mu_ld, n, c1r, c1i, c2r, c2i, C1r, C1i, C2r, C2i = _rexii_terms_ld(h, M)
    sel = n >= 0
    hh = LD(h)
    CL = np.clongdouble
    alpha = (hh * mu_ld) + 1j * CL(hh * n[sel].astype(LD))
    C1 = C1r[sel].astype(CL) + 1j * C1i[sel].astype(CL)
    C2 = C2r[sel].astype(CL) + 1j * C2i[sel].astype(CL)
    gamma = np.where(n[sel] == 0, LD(1), LD(2))
    return n[sel], alpha.astype(CL), C1, C2, gamma


@dataclass
class RexiTerms:
    """Term table of the original REXI, eq:originalRexi."""
    h: float
    M: int
    N: int
    n: np.ndarray
    alpha: np.ndarray
    beta_re: np.ndarray   # beta^{Re}_n = h sum a_k Re(b_{n-k})
    beta_im: np.ndarray   # beta^{Im}_n = h sum a_k Im(b_{n-k})


def rexi_terms(h, M):
    mu_ld, a_re, a_im = appendix_a(LD)
    L = L_APPENDIX_A
    N = M + L
    bre, bim = b_coeffs_ld(h, M)
    zb = np.zeros_like(bre)
    br_r, br_i = _windowed(h, M, L, a_re, a_im, bre, zb, N)   # a_k * Re(b)
    bi_r, bi_i = _windowed(h, M, L, a_re, a_im, bim, zb, N)   # a_k * Im(b)
    n = np.arange(-N, N + 1)
    hh = LD(h)
    alpha = float(hh * mu_ld) + 1j * (hh * n.astype(LD)).astype(np.float64)
    f = lambda r, i: r.astype(np.float64) + 1j * i.astype(np.float64)
    return RexiTerms(h=h, M=M, N=N, n=n, alpha=alpha, beta_re=f(br_r, br_i), beta_im=f(bi_r, bi_i))


# ---------------------------------------------------------------------------
# Scalar evaluators
# ---------------------------------------------------------------------------
def rexii_scalar(x, h, M, terms=None):
    """eq:modifiedRexi, PAPER.md:226-229:
    REXII(ix) = sum_{n=-N}^{N} (c_{1,n} h mu + c_{2,n}(x + h n)) / ((alpha_{-n} - ix)(alpha_n + ix))."""
    t = terms or rexii_terms(h, M)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    out = np.zeros(x.shape, dtype=np.complex128)
    alpha_minus = np.conj(t.alpha)   # alpha_{-n} = h(mu - i n)
    for j in range(len(t.n)):
        num = t.c1[j] * h * t.mu + t.c2[j] * (x + h * t.n[j])
        out += num / ((alpha_minus[j] - 1j * x) * (t.alpha[j] + 1j * x))
    return out


def rexi_scalar(x, h, M, terms=None):
    """eq:originalRexi, PAPER.md:211-214:
    REXI(ix) = sum_n Re(beta^Re_n/(ix + alpha_n)) + i Re(beta^Im_n/(ix + alpha_n))."""
    t = terms or rexi_terms(h, M)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    re = np.zeros(x.shape)
    im = np.zeros(x.shape)
    for j in range(len(t.n)):
        d = 1j * x + t.alpha[j]
        re += (t.beta_re[j] / d).real
        im += (t.beta_im[j] / d).real
    return re + 1j * im


# ---------------------------------------------------------------------------
# Term-count rule
# ---------------------------------------------------------------------------
def rho_lrsw(D):
    """eq:lswRoh, in the sqrt(2) pi D form of the Sec. 4.2 display
     — reading G5."""
    return math.sqrt(2.0) * math.pi * D


def m0_for_tol(tol, h):
    """Reading G9: the Appendix B construction applied
    to the shifted-Gaussian tail e^{h^2} psi_h((j+1)h) <= tol gives
    m0 = ceil(2 sqrt(h^2 - ln(sqrt(4 pi) tol)) - 1). At tol = 1e-16, h = 0.5 this is the
    paper's m0 = 11."""
    return int(math.ceil(2.0 * math.sqrt(h * h - math.log(math.sqrt(4.0 * math.pi) * tol)) - 1.0))


def h_for_tol(tol):
    """NEXT-2 h optimiser (readings G8, G9): largest h with e^{-4 pi (pi - h)} <= tol/10,
    clamped to [0.5, 2]."""
    if not (0.0 < tol < 1.0):
        return 0.5
    return min(2.0, max(0.5, math.pi - math.log(10.0 / tol) / (4.0 * math.pi)))


def M_rule(x_max, h, m0=11):
    """eq:Mformula / eq:matrixAccuracyBound: smallest M with x_max <= (M - m0) h."""
    return int(math.ceil(x_max / h)) + m0


def M_lrsw(D, tau, h, tol=None):
    """M for one LRSW step: tau*rho(A) <= (M - m0) h; m0 = 11 (paper) when tol is None."""
    m0 = 11 if tol is None else m0_for_tol(tol, h)
    return M_rule(abs(tau) * rho_lrsw(D), h, m0)


def half_sum_weights(h, M):
    """Per-pole data of eq:modifiedRexiMatrixReducedSum for n = 0..N:
    alpha_n, C_{1,n}, C_{2,n}, Gamma_n."""
    n, alpha, C1, C2, gamma = rexii_terms(h, M).half()
    return n, alpha, C1, C2, gamma
