"""GPU parity of ONE RANK'S SHARE of the poles (S3 + S4 building blocks) —
rexi_apply_partial and rexi_poles_real on the default in-contract PFHX kernel (and the others)
against the oracle's partial pole sum, element by element:

* full grids at 64^2 for every rank share of P = 2, 3, 8 (physical fields vs the oracle's
  dense-LU partial sum followed by its naive inverse DFT and Re);
* the full 512^2 grid for one rank's share of C2 on 8 GPUs (573 poles);
* 4096^2 (C4), the first and the last rank's share of 8 (4554 poles each), on sampled modes,
  against the oracle AND an extended-precision (long double) evaluation of the same partial
  sum: a partial sum cancels less than the full sum, so its fp64 rounding is larger; the
  tolerance is derived from the oracle's own distance to the long-double truth on the same
  modes (reading R1), not fitted to the GPU result.
"""
import numpy as np
import pytest

from oracle import coeffs as C
from oracle import lrsw
from paper_2008_11607_b200 import inputs
from paper_2008_11607_b200.distributed import pole_partition

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


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_partial_fields(f, tau, h, M, b, e):
    """Oracle: Re(IDFT(sum_{n in [b, e)} Gamma_n [...])) on the full grid (naive DFTs)."""
    D = f[0].shape[0]
    n, al, c1, c2, g = C.rexii_terms(h, M).half()
    F = lrsw.spectral_fields(*f)
    ml, mk = lrsw.all_modes(D)
    acc = lrsw.rexii_pole_sum(D, tau, F[ml, mk], ml, mk, al[b:e], c1[b:e], c2[b:e], g[b:e])
    A = np.zeros((D, D, 3), complex)
    A[ml, mk] = acc
    return np.stack([lrsw.idft2_real(A[..., c]) for c in range(3)])


@pytest.mark.parametrize("variant", ["pfhx", "pfhr", "pfh", "dz"])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_apply_partial_rank_shares_64(R, variant, P):
    D, tau, tol = 64, 1.0, 1e-12
    f = inputs.white_noise(D, seed=41)
    p = R.Plan(D, tau, tol=tol, variant=variant)
    info = p.info
    fd = [dev(x) for x in f]
    total = np.zeros((3, D, D))
    for r in range(P):
        b, e = pole_partition(p.n_poles, P, r)
        got = np.stack([host(t) for t in p.apply_partial(b, e, *fd)])
        ref = oracle_partial_fields(f, tau, info["h"], info["M"], b, e)
        assert rel(got, ref) < TOL, (r, rel(got, ref))
        total += got
    full = np.stack(lrsw.rexii_step(*f, tau, info["h"], info["M"]))
    assert rel(total, full) < TOL


def test_apply_partial_c2_rank_share_full_grid(R):
    """C2 (512^2, tau 1, tol 1e-8) split over 8 GPUs: rank 3's 573 poles, full grid."""
    D, tau, tol = 512, 1.0, 1e-8
    f = inputs.white_noise(D, seed=43)
    p = R.Plan(D, tau, tol=tol)
    info = p.info
    b, e = pole_partition(p.n_poles, 8, 3)
    got = np.stack([host(t) for t in p.apply_partial(b, e, *(dev(x) for x in f))])
    ref = oracle_partial_fields(f, tau, info["h"], info["M"], b, e)
    assert rel(got, ref) < TOL, rel(got, ref)


@pytest.mark.parametrize("variant", ["pfhx", "pfhr", "pfh"])
def test_poles_real_matches_hermitian_part_64(R, variant):
    """rexi_poles_real = the Hermitian part (A(K) + conj A(-K))/2 of the oracle's pole sum,
    full 64^2 grid, on pole sub-ranges; and rexi_inverse of it = rexi_apply_partial."""
    D, tau = 64, 1.0
    F = inputs.spectral_hermitian(D, seed=5)
    p = R.Plan(D, tau, variant=variant)
    n, al, c1, c2, g = C.rexii_terms(p.info["h"], p.info["M"]).half()
    ml, mk = lrsw.all_modes(D)
    mlm, mkm = (-ml) % D, (-mk) % D
    fm = np.stack([F[c][ml, mk] for c in range(3)], -1)
    fmm = np.stack([F[c][mlm, mkm] for c in range(3)], -1)
    for b, e in [(0, p.n_poles), (0, 1), (17, 140), (300, p.n_poles)]:
        acc = host(p.poles_real(dev(F), b, e))
        got = np.stack([acc[c][ml, mk] for c in range(3)], -1)
        s = slice(b, e)
        A = lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al[s], c1[s], c2[s], g[s])
        Am = lrsw.rexii_pole_sum(D, tau, fmm, mlm, mkm, al[s], c1[s], c2[s], g[s])
        assert rel(got, (A + np.conj(Am)) / 2) < TOL, (b, e)


@pytest.mark.parametrize("rank", [0, 7])
def test_poles_real_c4_rank_share_vs_oracle_and_long_double(R, rank):
    """4096^2, tau 1, tol 1e-12 (C4 on 8 GPUs): one rank's 4554 poles through the default PFHX
    kernel, 256 sampled modes (K = 0 modes, Nyquist lines and corners included).
    e_o = the fp64 oracle's distance to the long-double truth on these modes (what fp64 itself
    allows for this partial sum). Parity: GPU vs oracle < max(1e-12, 3 e_o); accuracy: GPU vs
    the truth < max(1e-12, 2 e_o) — the kernel is no less accurate than the dense-LU oracle."""
    D, tau, tol = 4096, 1.0, 1e-12
    p = R.Plan(D, tau, tol=tol)
    b, e = pole_partition(p.n_poles, 8, rank)
    F = inputs.spectral_hermitian(D, seed=9)
    ml, mk = inputs.sample_modes(D, 256)
    mlm, mkm = (-ml) % D, (-mk) % D
    fm = np.stack([F[c][ml, mk] for c in range(3)], -1)
    fmm = np.stack([F[c][mlm, mkm] for c in range(3)], -1)
    acc = p.poles_real(dev(F), b, e)
    del F
    got = np.stack([host(acc[c][ml, mk]) for c in range(3)], -1)
    del acc
    h, M = p.info["h"], p.info["M"]
    n, al, c1, c2, g = C.rexii_terms(h, M).half()
    s = slice(b, e)
    A = lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al[s], c1[s], c2[s], g[s])
    Am = lrsw.rexii_pole_sum(D, tau, fmm, mlm, mkm, al[s], c1[s], c2[s], g[s])
    ref = (A + np.conj(Am)) / 2
    tl = C.rexii_half_terms_ld(h, M)
    Ald = lrsw.rexii_pole_sum_ld(D, tau, fm, ml, mk, tl, b, e)
    Amld = lrsw.rexii_pole_sum_ld(D, tau, fmm, mlm, mkm, tl, b, e)
    truth = ((Ald + np.conj(Amld)) / 2).astype(np.complex128)
    e_o = rel(ref, truth)
    err = rel(got, ref)
    assert err < max(TOL, 3 * e_o), (err, e_o)
    assert rel(got, truth) < max(TOL, 2 * e_o), (rel(got, truth), e_o)
