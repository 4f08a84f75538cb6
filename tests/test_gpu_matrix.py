"""NEXT-3 on the GPU: the scalar forms per eigenvalue (rexi_scalar_apply) for the circulant test
matrices of Sec. 3.2 (diagonalised by the DFT in the test), against the oracle's dense-solve
matrix forms (parity) and expm (Fig. 2 behaviour)."""
import numpy as np
import pytest

from oracle import coeffs as C
from oracle import matrix as X

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def R():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2008_11607_b200 import build
    build.build()
    from paper_2008_11607_b200 import rexi
    return rexi


def gpu_apply(R, A, f, tau, h, M, method, nu=0.0):
    """The whole evaluation on the GPU through rexi_circulant_apply: the library's DFT kernels
    diagonalise the circulant A (eigenvalues = DFT of its first column), the scalar pole kernel
    applies r(tau (lambda - nu)) e^{tau nu} per eigenvalue, the inverse DFT returns the vector."""
    import torch
    col = torch.from_numpy(np.ascontiguousarray(A[:, 0].astype(np.complex128))).cuda()
    fd = torch.from_numpy(np.ascontiguousarray(f.astype(np.complex128))).cuda()
    sp = R.ScalarPlan(h, M)
    out = sp.circulant_apply(col, fd, tau, method=method, nu=nu)
    return out.cpu().numpy()


def test_scalar_rexii_vs_exp(R):
    """E2: at the minimal admissible M the scalar error is near machine precision
    for every x in the range; evaluated on the GPU for 4001 points."""
    import torch
    h, xmax = 0.5, 200.0
    M = C.M_rule(xmax, h)
    x = np.linspace(-xmax, xmax, 4001)
    sp = R.ScalarPlan(h, M)
    out = sp.apply(torch.from_numpy(x).cuda(), torch.ones(len(x), dtype=torch.complex128, device="cuda"))
    assert np.abs(out.cpu().numpy() - np.exp(1j * x)).max() < 1e-13
    # and the oracle's scalar REXII at a few points agrees to rounding. Tolerance (DESIGN.md
    # reading R3): two fp64 evaluations of the same n-term sum in different orders differ by
    # ~ sqrt(2n) u sum_n |term_n(x)| (random-walk rounding model, u = 2^-53), per point
    xs = x[::400]
    t = C.rexii_terms(h, M)
    am = np.conj(t.alpha)
    mag = np.zeros(len(xs))
    for j in range(len(t.n)):
        num = t.c1[j] * h * t.mu + t.c2[j] * (xs + h * t.n[j])
        mag += np.abs(num / ((am[j] - 1j * xs) * (t.alpha[j] + 1j * xs)))
    bound = np.sqrt(2 * len(t.n)) * 2.0 ** -53 * mag
    assert np.all(np.abs(out.cpu().numpy()[::400] - C.rexii_scalar(xs, h, M, terms=t)) < bound)


@pytest.mark.parametrize("h", [0.5, 0.2])
def test_fig2a_rexii_A1_gpu(R, h):
    A1, x = X.advection_A1()
    f = X.f0(x)
    M = C.M_rule(70.0, h)
    got = gpu_apply(R, A1, f, 1.0, h, M, "rexii")
    assert np.abs(got.imag).max() < 1e-12 * np.abs(got).max()
    ref = X.rexii_matrix(A1, f, 1.0, h, M)
    assert X.rel_l2(got.real, ref) < TOL
    assert X.rel_l2(got.real, X.expm_apply(A1, f, 1.0)) < 1e-13


@pytest.mark.parametrize("h", [0.5, 0.2])
def test_fig2b_rexi_A1_gpu(R, h):
    A1, x = X.advection_A1()
    f = X.f0(x)
    M = C.M_rule(70.0, h) + 10
    got = gpu_apply(R, A1, f, 1.0, h, M, "rexi_m").real     # eq:originalREXImatrix: Re of the vector
    ref = X.rexi_matrix(A1, f, 1.0, h, M)
    assert X.rel_l2(got, ref) < TOL
    assert X.rel_l2(got, X.expm_apply(A1, f, 1.0)) > 1e-7


def test_fig2c_rexie_A2_gpu(R):
    A2, x = X.schrodinger_A2()
    f = X.f0(x)
    M = C.M_rule(2450.0, 0.5)
    got = gpu_apply(R, A2, f, 1.0, 0.5, M, "rexi", nu=-2450j)
    ref = X.rexie_matrix(A2, f, 1.0, 0.5, M, nu=-2450j)
    assert X.rel_l2(got, ref) < TOL
    assert X.rel_l2(got, X.expm_apply(A2, f, 1.0)) < 1e-11


@pytest.mark.parametrize("n", [64, 70, 128])
def test_circulant_apply_transform_paths(R, n):
    """rexi_circulant_apply with both transform paths (Stockham passes for n = 64, 128; direct DFT
    for the paper's n = 70): REXII on A_1 vs the oracle's dense-solve matrix form and expm."""
    A1, x = X.advection_A1(n)
    f = X.f0(x)
    M = C.M_rule(float(n), 0.5)
    got = gpu_apply(R, A1, f, 1.0, 0.5, M, "rexii")
    assert np.abs(got.imag).max() < 1e-12 * np.abs(got).max()
    assert X.rel_l2(got.real, X.rexii_matrix(A1, f, 1.0, 0.5, M)) < TOL
    assert X.rel_l2(got.real, X.expm_apply(A1, f, 1.0)) < 1e-13
