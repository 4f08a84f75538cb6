"""The fused small-grid step (REXI_SCHEDULE_FUSED; AUTO picks it for small PFHX steps): the whole
S1..S5 as one launch of thread-block clusters exchanging stage data through distributed shared
memory (kernels.cu step_small2_kernel), element by element against the oracle on full grids,
including the pole range split over 1..8 clusters, pole sub-ranges (one rank's share), the REXI
method, graphs on/off and the host-buffer entry."""
import numpy as np
import pytest

from oracle import lrsw
from paper_2008_11607_b200 import inputs
from paper_2008_11607_b200.distributed import pole_partition

pytestmark = pytest.mark.gpu
TOL = 1e-12
FUSED = 3


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
    a = np.concatenate([np.ravel(x) for x in a])
    b = np.concatenate([np.ravel(x) for x in b])
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("D,tau,tol,scen", [(4, 0.5, 1e-12, "white"), (8, 0.7, 1e-12, "white"),
                                            (16, 1.0, 1e-12, "white"), (32, 3.0, 1e-10, "white"),
                                            (64, 0.02, 1e-12, "gauss"), (64, 0.02, 1e-12, "white"),
                                            (64, 1.0, 1e-12, "white"), (128, 0.05, 1e-12, "white"),
                                            (128, 1.0, 1e-12, "gauss")])
def test_fused_step_vs_oracle(R, D, tau, tol, scen, graphs):
    f = inputs.gaussian_scenario(D) if scen == "gauss" else inputs.white_noise(D, seed=71)
    p = R.Plan(D, tau, tol=tol)
    p.set_schedule("fused")
    p.set_graphs(graphs)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    assert p.info["last_schedule"] == FUSED
    info = p.info
    ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
    assert rel(got, ref) < TOL
    # and the multi-launch path agrees to summation order
    q = R.Plan(D, tau, tol=tol)
    q.set_schedule("chunked")
    other = [host(t) for t in q.apply(*(dev(x) for x in f))]
    assert rel(got, other) < 1e-13


@pytest.mark.parametrize("clusters", [1, 2, 3, 8])
@pytest.mark.parametrize("D,tau,scen", [(4, 0.5, "white"), (16, 1.0, "white"), (64, 0.02, "gauss"),
                                        (64, 1.0, "white"), (128, 0.05, "white")])
def test_fused_clusters_vs_oracle(R, D, tau, scen, clusters):
    """The pole range split over `clusters` clusters (partial spectra summed by the last cluster
    to finish, in cluster order) against the oracle; repeated launches reuse the arrival counter."""
    f = inputs.gaussian_scenario(D) if scen == "gauss" else inputs.white_noise(D, seed=77)
    p = R.Plan(D, tau, tol=1e-12)
    p.set_schedule("fused")
    p.set_fused_clusters(clusters)
    fd = [dev(x) for x in f]
    info = p.info
    ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
    first = [host(t) for t in p.apply(*fd)]
    assert p.info["last_schedule"] == FUSED
    assert rel(first, ref) < TOL
    for _ in range(3):
        again = [host(t) for t in p.apply(*fd)]
    for x, y in zip(first, again):
        assert np.array_equal(x, y)   # fixed summation order: bit-for-bit across launches


def test_fused_clusters_rejects_out_of_range(R):
    p = R.Plan(16, 0.5, tol=1e-12)
    for bad in (-1, 10):
        with pytest.raises(R.RexiError):
            p.set_fused_clusters(bad)


def test_auto_picks_fused_for_c1(R):
    """C1 (64^2, tau 0.02, 47 poles): AUTO runs the fused step (one launch per step)."""
    D, tau = 64, 0.02
    f = [dev(x) for x in inputs.gaussian_scenario(D)]
    p = R.Plan(D, tau, tol=1e-12)
    p.apply(*f)
    assert p.info["last_schedule"] == FUSED
    p.timing_enable(True)
    p.timing_read()
    for _ in range(3):
        p.apply(*f)
    ms, pl, tl = p.timing_read()
    assert pl == 3 and tl == 3 and ms > 0
    # large pole work stays on the chunked path under AUTO
    big = R.Plan(128, 1.0, tol=1e-12)
    big.apply(*(dev(x) for x in inputs.white_noise(128)))
    assert big.info["last_schedule"] == 1


@pytest.mark.parametrize("P", [2, 3, 8])
def test_fused_apply_partial_vs_oracle(R, P):
    """One rank's share through the fused step vs the oracle's partial sum (full 64^2 grid)."""
    from oracle import coeffs as C
    D, tau = 64, 1.0
    f = inputs.white_noise(D, seed=73)
    p = R.Plan(D, tau, tol=1e-12)
    p.set_schedule("fused")
    info = p.info
    n, al, c1, c2, g = C.rexii_terms(info["h"], info["M"]).half()
    F = lrsw.spectral_fields(*f)
    ml, mk = lrsw.all_modes(D)
    fd = [dev(x) for x in f]
    for r in range(P):
        b, e = pole_partition(p.n_poles, P, r)
        got = np.stack([host(t) for t in p.apply_partial(b, e, *fd)])
        acc = lrsw.rexii_pole_sum(D, tau, F[ml, mk], ml, mk, al[b:e], c1[b:e], c2[b:e], g[b:e])
        A = np.zeros((D, D, 3), complex)
        A[ml, mk] = acc
        ref = np.stack([lrsw.idft2_real(A[..., c]) for c in range(3)])
        assert rel(got, ref) < TOL, (r, rel(got, ref))


def test_fused_rexi_method_and_host(R):
    from oracle import coeffs as C  # noqa: F401
    D, tau, h, M = 32, 1.0, 0.2, 200
    f = inputs.white_noise(D, seed=75)
    p = R.Plan(D, tau, h=h, M=M, method="rexi")
    p.set_schedule("fused")
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    ref = lrsw.rexi_step(*f, tau, h, M)
    assert rel(got, ref) < TOL
    import torch
    q = R.Plan(64, 0.02, tol=1e-12)
    g = inputs.gaussian_scenario(64)
    out = q.apply_host(*[torch.from_numpy(np.ascontiguousarray(x)) for x in g])
    ref = lrsw.rexii_step(*g, 0.02, q.info["h"], q.info["M"])
    assert q.info["last_schedule"] == FUSED
    assert rel(list(out), ref) < TOL


@pytest.mark.parametrize("D,tau,K", [(8, 0.3, 3), (16, 0.2, 4), (64, 0.02, 5)])
def test_fused_run_vs_oracle_steps(R, D, tau, K):
    """rexi_run on a small grid: the whole K-step run as one fused launch (the state stays in the
    cluster's shared memory between steps) against K oracle steps, and against K single steps."""
    import torch
    f = inputs.white_noise(D, seed=79)
    p = R.Plan(D, tau, tol=1e-12)
    info = p.info
    ref = f
    for _ in range(K):
        ref = lrsw.rexii_step(*ref, tau, info["h"], info["M"])
    x = [dev(a) for a in f]
    p.timing_enable(True)
    p.timing_read()
    p.run(K, *x)
    ms, pl, tl = p.timing_read()
    assert tl == 1 and p.info["last_schedule"] == FUSED   # one launch for the whole run
    got = [host(t) for t in x]
    assert rel(got, ref) < K * TOL
    y = [dev(a) for a in f]
    for _ in range(K):
        y = [t.clone() for t in p.apply(*y)]
    assert rel(got, [host(t) for t in y]) < 1e-13
