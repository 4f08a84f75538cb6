"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element on the
same seeded inputs. Tolerance (north_star): relative L2 <= 1e-12 in fp64 with identical
coefficients (the planner's and the oracle's tables agree to ~1e-15, test_capi_host.py)."""
import math

import numpy as np
import pytest

from oracle import coeffs as C
from oracle import lrsw
from paper_2008_11607_b200 import inputs

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


def rel_l2(a, b):
    a = np.concatenate([np.ravel(x) for x in a])
    b = np.concatenate([np.ravel(x) for x in b])
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_terms(plan):
    h, M = plan.info["h"], plan.info["M"]
    return C.rexii_terms(h, M)


# ----------------------------------------------------------------------------- S0
def test_plan_coeffs_match_oracle(R):
    p = R.Plan(512, 1.0, tol=1e-8)
    assert p.info["M"] == 4558 and p.n_poles == 4583
    al, c1, c2, g = p.coeffs()
    n, oal, oc1, oc2, og = oracle_terms(p).half()
    s = np.abs(oc1).max()
    assert np.abs(al - oal).max() < 1e-14 * np.abs(oal).max()
    assert np.abs(c1 - oc1).max() < 2e-15 * s and np.abs(c2 - oc2).max() < 2e-15 * s
    assert np.array_equal(g, og)


def test_plan_errors(R):
    with pytest.raises(R.RexiError):
        R.Plan(100, 1.0)                # not a power of two
    with pytest.raises(R.RexiError):
        R.Plan(64, 1.0, h=3.5)
    with pytest.raises(R.RexiError):
        R.Plan(64, float("nan"))
    with pytest.raises(R.RexiError):
        R.Plan(64, 1.0, M=5)
    p = R.Plan(16, 0.1)
    import torch
    f = torch.zeros((3, 16, 16), dtype=torch.complex128, device="cuda")
    with pytest.raises(R.RexiError):
        p.poles(f, 0, p.n_poles + 1)
    with pytest.raises(R.RexiError):
        p.poles(f, 5, 4)
    with pytest.raises(ValueError):
        p.apply(*(torch.zeros((8, 8), dtype=torch.float64, device="cuda") for _ in range(3)))


# ----------------------------------------------------------------------------- S1 / S5
@pytest.mark.parametrize("D", [4, 8, 16, 32, 64, 128, 256, 512, 1024])
def test_forward_fft_vs_naive_dft(R, D):
    p = R.Plan(D, 0.1)
    f = inputs.white_noise(D)
    F = host(p.forward(*(dev(x) for x in f)))
    import torch
    torch.cuda.synchronize()
    for c in range(3):
        O = lrsw.dft2(f[c])
        assert np.linalg.norm(F[c] - O) / np.linalg.norm(O) < 1e-14


@pytest.mark.parametrize("D", [4, 8, 16, 32, 64, 256, 512, 1024])
def test_inverse_fft_vs_naive_dft(R, D):
    p = R.Plan(D, 0.1)
    A = inputs.spectral_white(D, seed=3)
    out = [host(t) for t in p.inverse(dev(A))]
    for c in range(3):
        O = lrsw.idft2_real(A[c])
        assert np.linalg.norm(out[c] - O) / np.linalg.norm(O) < 1e-14


def test_fft_4096_sampled(R):
    """Full C4 grid size: sampled entries of the forward transform vs the DFT definition."""
    D = 4096
    p = R.Plan(D, 1.0, tol=1e-12)
    g = np.random.Generator(np.random.PCG64(1))
    X = g.standard_normal((D, D))
    import torch
    Z = torch.zeros((D, D), dtype=torch.float64, device="cuda")
    F = p.forward(dev(X), Z, Z)
    F0 = host(F[0])
    x = np.arange(D)
    for (l, k) in [(0, 0), (1, 0), (0, 2048), (2048, 2048), (17, 4095), (3000, 1234)]:
        ph = np.exp(-2j * np.pi * ((k * x[None, :] + l * x[:, None]) % D) / D)
        ref = (X * ph).sum() / D ** 2
        assert abs(F0[l, k] - ref) < 1e-13 * np.sqrt(D * D) / D ** 2 * 50


@pytest.mark.parametrize("D", [2048, 8192])
def test_fft_sampled_and_round_trip_large(R, D):
    """The radix-16 passes at the sizes no full-grid test covers: sampled entries of the forward
    transform and of the (symmetrising) inverse vs the DFT definition, and inverse(forward(X))
    = X for real X over the whole grid."""
    import torch
    p = R.Plan(D, 0.001, tol=1e-8)
    g = np.random.Generator(np.random.PCG64(D))
    X = g.standard_normal((D, D))
    Z = torch.zeros((D, D), dtype=torch.float64, device="cuda")
    Xd = dev(X)
    F = p.forward(Xd, Z, Z)
    F0 = host(F[0])
    x = np.arange(D)
    H = D // 2
    for (l, k) in [(0, 0), (1, 0), (0, H), (H, H), (17, D - 1), (D - 5, 3)]:
        ph = np.exp(-2j * np.pi * ((k * x[None, :] + l * x[:, None]) % D) / D)
        ref = (X * ph).sum() / D ** 2
        assert abs(F0[l, k] - ref) < 1e-13 * np.sqrt(D * D) / D ** 2 * 50
    back = [host(t) for t in p.inverse(F)]
    assert np.abs(back[0] - X).max() < 1e-12
    assert np.abs(back[1]).max() < 1e-12 and np.abs(back[2]).max() < 1e-12
    # inverse of a non-Hermitian spectrum (symmetrised on load) at sampled points
    A = torch.zeros_like(F)
    A[0] = F[0] * (1.0 + 0.5j)             # breaks the Hermitian symmetry
    out0 = host(p.inverse(A)[0])
    Ah = host(A[0])
    for (yy, xx) in [(0, 0), (3, D - 2), (H, 7)]:
        ph = np.exp(2j * np.pi * ((xx * x[None, :] + yy * x[:, None]) % D) / D)
        assert abs(out0[yy, xx] - (Ah * ph).sum().real) < 1e-11


# ----------------------------------------------------------------------------- S2 + S3
def _pole_parity(R, D, tau, tol, variant, modes=None, begin=0, end=None, seed=5):
    p = R.Plan(D, tau, tol=tol, variant=variant)
    end = p.n_poles if end is None else end
    F = inputs.spectral_white(D, seed=seed)
    acc = host(p.poles(dev(F), begin, end))
    n, al, c1, c2, gm = oracle_terms(p).half()
    if modes is None:
        ml, mk = lrsw.all_modes(D)
    else:
        ml, mk = modes
    fm = np.stack([F[c][ml, mk] for c in range(3)], axis=-1)
    ref = lrsw.rexii_pole_sum(D, tau, fm, ml, mk, al[begin:end], c1[begin:end], c2[begin:end],
                              gm[begin:end])
    got = np.stack([acc[c][ml, mk] for c in range(3)], axis=-1)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    # per-mode check too: each sampled mode within 1e-11 relative of its own magnitude
    pm = np.linalg.norm(got - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
    return err, float(pm.max())


@pytest.mark.parametrize("variant", ["dz", "uv", "dz3", "pf", "pfh"])
@pytest.mark.parametrize("D,tau,tol", [(4, 0.5, 1e-12), (8, 1.0, 1e-12), (64, 0.02, 1e-12),
                                       (64, 1.0, 1e-12), (32, 5.0, 1e-8)])
def test_pole_kernel_full_grid(R, variant, D, tau, tol):
    err, pm = _pole_parity(R, D, tau, tol, variant)
    assert err < TOL, err
    assert pm < 1e-11, pm


@pytest.mark.parametrize("variant", ["dz", "uv", "dz3", "pf", "pfh"])
def test_pole_kernel_ranges(R, variant):
    D, tau = 64, 1.0
    for (b, e) in [(0, 1), (1, 2), (0, 37), (100, 333), (500, 604)]:
        err, pm = _pole_parity(R, D, tau, 1e-12, variant, begin=b, end=e)
        assert err < TOL, (b, e, err)


def test_pole_kernel_empty_range_is_zero(R):
    p = R.Plan(16, 1.0)
    import torch
    F = dev(inputs.spectral_white(16))
    acc = p.poles(F, 7, 7)
    assert float(acc.abs().max()) == 0.0


@pytest.mark.parametrize("variant", ["dz", "uv", "dz3", "pf", "pfh"])
def test_pole_kernel_c2_full_size_sampled(R, variant):
    """BASELINE configs[1] (512^2, tau = 1, tol 1e-8, 4583 poles) in the launch configuration
    bench.py times; 2048 sampled modes incl. K = 0, Nyquist row/column and the corner."""
    modes = inputs.sample_modes(512, 2048)
    err, pm = _pole_parity(R, 512, 1.0, 1e-8, variant, modes=modes)
    assert err < TOL, err
    assert pm < 1e-11, pm


@pytest.mark.parametrize("variant", ["dz", "dz3", "pf", "pfh"])
def test_pole_kernel_c4_size_sampled(R, variant):
    """4096^2 grid, tau = 1, tol 1e-12 (configs[3]): all 36432 poles, 512 sampled modes.
    (A pole SUB-range is a harder target: its terms cancel less, and the independent fp64
    roundings of the two sides' per-pole constants (~1e-16 relative) show up at ~1e-12 relative
    of the partial sum — DESIGN.md "Precision". The full sum is the configuration's step.)"""
    modes = inputs.sample_modes(4096, 512)
    err, pm = _pole_parity(R, 4096, 1.0, 1e-12, variant, modes=modes)
    assert err < TOL, err


# ----------------------------------------------------------------------------- S1..S5
@pytest.mark.parametrize("variant", ["dz", "uv", "dz3", "pf", "pfh", "pfhr", "pfhx"])
@pytest.mark.parametrize("D,tau,tol,scen", [(64, 0.02, 1e-12, "gauss"), (64, 0.02, 1e-12, "white"),
                                            (128, 1.0, 1e-12, "gauss"), (32, 3.0, 1e-10, "white"),
                                            (8, 0.7, 1e-12, "white")])
def test_apply_vs_oracle(R, variant, D, tau, tol, scen):
    f = inputs.gaussian_scenario(D) if scen == "gauss" else inputs.white_noise(D)
    p = R.Plan(D, tau, tol=tol, variant=variant)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    info = p.info
    ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
    assert rel_l2(got, ref) < TOL
    ex = lrsw.exact_step(*f, tau)
    assert rel_l2(got, ex) < max(tol, 1e-13)


def test_apply_c2_full_size_properties(R):
    """Full C2 (512^2, tau=1, tol=1e-8), Gaussian scenario: vs the exact per-mode propagator
    within tol, energy conservation and mean(eta) conservation."""
    D = 512
    f = inputs.gaussian_scenario(D)
    p = R.Plan(D, 1.0, tol=1e-8)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    ex = lrsw.exact_step(*f, 1.0)
    assert rel_l2(got, ex) < 1e-8
    e0 = sum(float((x ** 2).sum()) for x in f)
    e1 = sum(float((x ** 2).sum()) for x in got)
    assert abs(e1 - e0) / e0 < 1e-8
    assert abs(got[0].mean() - f[0].mean()) < 1e-13


def test_apply_partial_partition_invariance(R):
    """S4 on one GPU: sum over a pole partition of rexi_apply_partial == rexi_apply."""
    from paper_2008_11607_b200.distributed import pole_partition
    D = 64
    f = [dev(x) for x in inputs.white_noise(D)]
    p = R.Plan(D, 1.0)
    full = [host(t) for t in p.apply(*f)]
    for P in (2, 3, 8):
        tot = [np.zeros((D, D)) for _ in range(3)]
        for r in range(P):
            b, e = pole_partition(p.n_poles, P, r)
            part = p.apply_partial(b, e, *f)
            for c in range(3):
                tot[c] += host(part[c])
        assert rel_l2(tot, full) < 1e-14


def test_apply_in_place_and_host_and_run(R):
    import torch
    D, tau = 32, 0.4
    f = inputs.white_noise(D)
    p = R.Plan(D, tau)
    ref = [host(t) for t in p.apply(*(dev(x) for x in f))]
    # host-buffer entry
    hout = p.apply_host(*(np.ascontiguousarray(x) for x in f))
    assert rel_l2(hout, ref) == 0.0
    # in place
    t = [dev(x) for x in f]
    p.apply(*t, out=t)
    assert rel_l2([host(x) for x in t], ref) == 0.0
    # multi-step driver (S6): 3 steps vs 3 oracle steps
    t = [dev(x) for x in f]
    p.run(3, *t)
    g = f
    info = p.info
    terms = C.rexii_terms(info["h"], info["M"])
    for _ in range(3):
        g = lrsw.rexii_step(*g, tau, info["h"], info["M"], terms=terms)
    assert rel_l2([host(x) for x in t], g) < TOL


@pytest.mark.parametrize("batch", [1, 2, 5])
def test_apply_host_batch(R, batch):
    """rexi_apply_host_batch: problem i of the batch equals rexi_apply on it (same kernels,
    bit-identical), for numpy and pinned-tensor host buffers; one problem checked vs the oracle."""
    import torch
    D, tau = 32, 0.4
    p = R.Plan(D, tau)
    fs = [inputs.white_noise(D, seed=100 + 10 * i) for i in range(batch)]
    stack = [np.ascontiguousarray(np.stack([f[c] for f in fs])) for c in range(3)]
    out = p.apply_host_batch(*stack)
    for i, f in enumerate(fs):
        ref = [host(t) for t in p.apply(*(dev(x) for x in f))]
        assert rel_l2([o[i] for o in out], ref) == 0.0
    pin = [torch.from_numpy(x).pin_memory() for x in stack]
    pout = [torch.empty_like(x).pin_memory() for x in pin]
    p.apply_host_batch(*pin, out=pout)
    for c in range(3):
        assert np.array_equal(pout[c].numpy(), out[c])
    info = p.info
    g = lrsw.rexii_step(*fs[-1], tau, info["h"], info["M"])
    assert rel_l2([o[-1] for o in out], g) < TOL


def test_apply_host_batch_errors(R):
    p = R.Plan(8, 0.3)
    z = np.zeros((2, 8, 8))
    with pytest.raises(ValueError):
        p.apply_host_batch(z, z, np.zeros((3, 8, 8)))
    with pytest.raises(ValueError):
        p.apply_host_batch(z, z, np.zeros((2, 8, 4)))
    out = p.apply_host_batch(z[:0], z[:0], z[:0])
    assert out[0].shape == (0, 8, 8)


@pytest.mark.parametrize("D,tau,tol", [(64, 1.0, 1e-12), (128, 1.0, 1e-12), (128, 3.0, 1e-8),
                                       (256, 0.5, 1e-12)])
def test_schedules_agree(R, D, tau, tol):
    """Stream-K and chunked R2C pole schedules: same result up to summation order; stream-K vs
    the oracle on the smaller cases; AUTO runs the chunked schedule."""
    import torch
    f = inputs.white_noise(D, seed=5)
    fd = [dev(x) for x in f]
    res = {}
    for sched in ("chunked", "streamk", "auto"):
        p = R.Plan(D, tau, tol=tol, variant="pfhr")   # stream-K exists for the PFHR kernel only
        p.set_schedule(sched)
        res[sched] = [host(t) for t in p.apply(*fd)]
        info = p.info
        res[sched + "_used"] = info["last_schedule"]
    assert res["chunked_used"] == 1 and res["auto_used"] == 1
    assert res["streamk_used"] == 2
    assert rel_l2(res["streamk"], res["chunked"]) < 1e-14
    assert rel_l2(res["auto"], res["chunked"]) < 1e-14
    if D <= 128:
        info = R.Plan(D, tau, tol=tol, variant="pfhr").info
        g = lrsw.rexii_step(*f, tau, info["h"], info["M"])
        assert rel_l2(res["streamk"], g) < TOL


def test_schedule_errors(R):
    p = R.Plan(16, 0.3)
    with pytest.raises(ValueError):
        p.set_schedule("dynamic")
    assert p.info["schedule"] == 0 and p.info["last_schedule"] == 0


@pytest.mark.parametrize("spectral", [False, True])
@pytest.mark.parametrize("variant", ["pfhx", "pfh"])
def test_run_distributed_single_rank_matches_run(R, spectral, variant):
    """distributed.run_distributed (per-step pole split + all-reduce; one rank here), in
    physical or spectral-resident form, equals rexi_run up to rounding, and the oracle's steps."""
    from paper_2008_11607_b200.distributed import run_distributed
    D, tau = 32, 0.7
    f = inputs.white_noise(D, seed=31)
    p = R.Plan(D, tau, variant=variant)
    a = [dev(x) for x in f]
    b = [dev(x) for x in f]
    p.run(3, *a)
    run_distributed(p, 3, *b, spectral=spectral)
    assert rel_l2([host(x) for x in b], [host(x) for x in a]) < 1e-13
    g = f
    for _ in range(3):
        g = lrsw.rexii_step(*g, tau, p.info["h"], p.info["M"])
    assert rel_l2([host(x) for x in b], g) < TOL


@pytest.mark.parametrize("D", [4, 8, 64])
def test_hermitian_mirror(R, D):
    """rexi_hermitian_mirror rebuilds rows D/2+1 .. D-1 of a Hermitian spectrum exactly and
    leaves rows 0 .. D/2 untouched."""
    import torch
    F = inputs.spectral_hermitian(D, seed=2)
    p = R.Plan(D, 0.5)
    t = dev(F)
    t[:, D // 2 + 1:] = 0
    got = host(p.hermitian_mirror(t))
    assert np.array_equal(got, F)


def test_variants_agree(R):
    D = 128
    f = [dev(x) for x in inputs.white_noise(D)]
    res = {}
    for v in ("dz", "uv", "dz3", "pf", "pfh", "pfhr", "pfhx"):
        res[v] = [host(t) for t in R.Plan(D, 2.0, variant=v).apply(*f)]
    for v in ("uv", "dz3", "pf", "pfh", "pfhr", "pfhx"):
        assert rel_l2(res["dz"], res[v]) < TOL


def test_timing_counters(R):
    D = 64
    f = [dev(x) for x in inputs.white_noise(D)]
    p = R.Plan(D, 1.0)
    p.set_schedule("chunked")             # seven launches per step
    p.timing_enable(True)
    p.timing_read()
    for _ in range(3):
        p.apply(*f)
    ms, pl, tl = p.timing_read()
    assert pl == 3 and ms > 0.0 and tl == 3 * 7
    p.set_schedule("auto")                # 64^2, 604 poles: the fused step, one launch per step
    for _ in range(3):
        p.apply(*f)
    ms, pl, tl = p.timing_read()
    assert pl == 3 and ms > 0.0 and tl == 3


TUNINGS = [("dz", 1, 1, 8), ("dz", 2, 1, 4), ("dz", 2, 1, 5), ("dz", 3, 1, 4), ("dz", 4, 1, 3),
           ("dz", 4, 1, 4),
           ("uv", 1, 1, 6), ("uv", 2, 1, 3), ("uv", 2, 1, 4), ("uv", 3, 1, 3), ("uv", 4, 1, 2),
           ("uv", 4, 1, 3),
           ("dz3", 1, 1, 8), ("dz3", 2, 1, 4), ("dz3", 3, 1, 4), ("dz3", 4, 1, 2), ("dz3", 4, 1, 4),
           ("pf", 1, 1, 8), ("pf", 2, 1, 3), ("pf", 2, 1, 4), ("pf", 3, 1, 4), ("pf", 4, 1, 3),
           ("pf", 4, 1, 4),
           ("pfh", 1, 1, 8), ("pfh", 2, 1, 3), ("pfh", 2, 1, 4), ("pfh", 3, 1, 4), ("pfh", 4, 1, 3),
           ("pfh", 4, 1, 4), ("pfh", 1, 2, 6), ("pfh", 2, 2, 3), ("pfh", 2, 2, 4), ("pfh", 4, 2, 2)]


@pytest.mark.parametrize("variant,mpt,pu,minb", TUNINGS)
def test_pole_kernel_tunings(R, variant, mpt, pu, minb):
    """Every pole-kernel instantiation gives the same result up to the summation order of the
    pole chunks (the chunk count follows the tile count) and matches the oracle (ragged tails: D = 32 has 1024 modes, not a multiple of 384 at mpt 3 or 512 at
    mpt 4; D = 8 has one partial tile)."""
    for D in (8, 32):
        p = R.Plan(D, 1.3, variant=variant)
        F = dev(inputs.spectral_white(D, seed=9))
        base = host(p.poles(F))
        p.set_tuning(mpt, pu, minb)
        acc = host(p.poles(F))
        assert np.linalg.norm(acc - base) <= 1e-14 * np.linalg.norm(base)
        n, al, c1, c2, gm = oracle_terms(p).half()
        ml, mk = lrsw.all_modes(D)
        Fh = host(F)
        fm = np.stack([Fh[c][ml, mk] for c in range(3)], axis=-1)
        ref = lrsw.rexii_pole_sum(D, 1.3, fm, ml, mk, al, c1, c2, gm)
        got = np.stack([acc[c][ml, mk] for c in range(3)], axis=-1)
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < TOL


def test_tuning_rejects_unsupported(R):
    p = R.Plan(16, 1.0)
    with pytest.raises(R.RexiError):
        p.set_tuning(3, 3, 3)



# ----------------------------------------------------------------------------- paper rows on GPU
from conftest import read_paper_tables  # noqa: E402

_SCEN = {"wave1": inputs.wave_scenario_1, "wave2": inputs.wave_scenario_2,
         "gaussian": inputs.gaussian_scenario}

# The printed rows of tests/golden/paper_tables.txt plus the large-M rows of Tables 3, 4, 6, 7
# (too slow for the CPU oracle on the full grid; one GPU step each here).
EXTRA_ROWS = [
    dict(method="REXII", scenario="wave1", tau=50.0, h=0.1, M=13341, paper=1.81e-13, cite="PAPER.md:664"),
    dict(method="REXII", scenario="wave2", tau=50.0, h=0.5, M=56885, paper=6.53e-13, cite="PAPER.md:706"),
    dict(method="REXII", scenario="wave2", tau=50.0, h=0.1, M=284371, paper=9.36e-13, cite="PAPER.md:707"),
    dict(method="REXII", scenario="gaussian", tau=1.0, h=0.1, M=5698, paper=1.53e-14, cite="PAPER.md:764"),
    dict(method="REXII", scenario="gaussian", tau=50.0, h=1.0, M=28448, paper=6.18e-13, cite="PAPER.md:787"),
    dict(method="REXII", scenario="gaussian", tau=50.0, h=0.5, M=56885, paper=6.06e-14, cite="PAPER.md:788"),
    dict(method="REXII", scenario="gaussian", tau=50.0, h=0.1, M=284371, paper=1.04e-13, cite="PAPER.md:789"),
    dict(method="REXI", scenario="wave1", tau=1.0, h=0.2, M=100000, paper=3.27e-8, cite="PAPER.md:629"),
    dict(method="REXI", scenario="gaussian", tau=1.0, h=0.2, M=1500, paper=3.78e-4, cite="PAPER.md:758"),
    dict(method="REXI", scenario="gaussian", tau=1.0, h=0.2, M=3000, paper=3.21e-6, cite="PAPER.md:759"),
]


@pytest.mark.parametrize("row", read_paper_tables() + EXTRA_ROWS,
                         ids=lambda r: f"{r['method']}-{r['scenario']}-t{r['tau']}-h{r['h']}-M{r['M']}")
def test_gpu_reproduces_paper_rows(R, row):
    """The CUDA path's one-step max-norm error vs the exact propagator (reading G15) on the
    paper's 128^2 grid reproduces each printed error within a factor 2.5 (Tables 2-7)."""
    D = 128
    f = _SCEN[row["scenario"]](D)
    p = R.Plan(D, row["tau"], h=row["h"], M=row["M"], method=row["method"].lower())
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    ex = lrsw.exact_step(*f, row["tau"])
    err = max(float(np.abs(a - b).max()) for a, b in zip(got, ex))
    assert row["paper"] / 2.5 < err < row["paper"] * 2.5, (err, row)


@pytest.mark.parametrize("D,tau,h,M", [(16, 1.0, 0.2, 150), (32, 0.5, 0.2, 400), (8, 2.0, 0.5, 60)])
def test_rexi_method_vs_oracle(R, D, tau, h, M):
    """NEXT-1: the original REXI on the GPU (half-sum, reading R2) vs the oracle's full sum
    n = -N..N of eq:originalREXImatrix with dense solves, after Re."""
    f = inputs.white_noise(D)
    p = R.Plan(D, tau, h=h, M=M, method="rexi")
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    ref = lrsw.rexi_step(*f, tau, h, M)
    assert rel_l2(got, ref) < TOL


@pytest.mark.parametrize("variant", ["uv", "dz", "dz3", "pf", "pfh", "pfhr", "pfhx"])
@pytest.mark.parametrize("D,tau,h,M", [(16, 1.0, 0.2, 150), (64, 0.5, 0.2, 500)])
def test_rexi_method_variants(R, variant, D, tau, h, M):
    """REXI (w2 = 0) through every variant: the DZ back-substitution kernel (uv, dz, dz3) and
    the partial-fraction kernels with W1 = w1, W2 = 0 (pf, pfh, pfhr, pfhx incl. R2C octets)."""
    f = inputs.white_noise(D, seed=21)
    p = R.Plan(D, tau, h=h, M=M, method="rexi", variant=variant)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    ref = lrsw.rexi_step(*f, tau, h, M)
    assert rel_l2(got, ref) < TOL


@pytest.mark.parametrize("mpt,pu,minb", [(1, 1, 8), (2, 1, 4), (4, 1, 4), (4, 1, 5)])
def test_rexi_method_tunings(R, mpt, pu, minb):
    D, tau, h, M = 32, 1.0, 0.2, 300
    f = [dev(x) for x in inputs.white_noise(D)]
    p = R.Plan(D, tau, h=h, M=M, method="rexi", variant="dz")
    base = [host(t) for t in p.apply(*f)]
    p.set_tuning(mpt, pu, minb)
    got = [host(t) for t in p.apply(*f)]
    assert rel_l2(got, base) < 1e-14


def test_set_method_invalidates_graphs(R):
    """apply (REXII) -> set_method('rexi') -> apply into the SAME buffers must not replay the
    REXII graph (its finish / fix-up arguments carry the old method's pole sums): the result
    equals a fresh REXI plan's, and switching back reproduces the REXII result."""
    import torch
    D, tau, h, M = 32, 1.0, 0.2, 200
    f = [dev(x) for x in inputs.white_noise(D, seed=77)]
    out = [torch.empty((D, D), dtype=torch.float64, device="cuda") for _ in range(3)]
    for variant in ("pfhx", "pfhr", "pfh", "dz"):
        p = R.Plan(D, tau, h=h, M=M, variant=variant)
        a = [host(t) for t in p.apply(*f, out=out)]
        p.set_method("rexi")
        b = [host(t) for t in p.apply(*f, out=out)]
        ref = [host(t) for t in R.Plan(D, tau, h=h, M=M, method="rexi", variant=variant).apply(*f)]
        assert rel_l2(b, ref) == 0.0, variant
        p.set_method("rexii")
        c = [host(t) for t in p.apply(*f, out=out)]
        assert rel_l2(c, a) == 0.0, variant
        assert rel_l2(b, a) > 1e-6          # the two methods really differ at this (h, M)


def test_set_method_roundtrip(R):
    D = 32
    f = [dev(x) for x in inputs.white_noise(D)]
    p = R.Plan(D, 1.0, h=0.2, M=200)
    a = [host(t) for t in p.apply(*f)]
    p.set_method("rexi")
    al, beta, zero, g = p.coeffs()
    assert np.all(zero == 0)
    p.set_method("rexii")
    b = [host(t) for t in p.apply(*f)]
    assert rel_l2(a, b) == 0.0
    assert p.info["method"] == 0


def test_graphs_match_direct_and_timing(R):
    """Whole-step CUDA graphs: identical results to direct launches; the timing events inside
    a replayed graph are re-targeted per replay (one pole-kernel interval per step)."""
    D = 64
    f = [dev(x) for x in inputs.white_noise(D)]
    p = R.Plan(D, 1.0)
    p.set_schedule("chunked")             # the seven-launch graph (AUTO fuses 64^2 steps)
    p.set_graphs(False)
    a = [host(t) for t in p.apply(*f)]
    p.set_graphs(True)
    for _ in range(2):
        b = [host(t) for t in p.apply(*f)]
        assert rel_l2(b, a) == 0.0
    p.timing_enable(True)
    p.timing_read()
    for _ in range(4):
        p.apply(*f)
    ms, pl, tl = p.timing_read()
    assert pl == 4 and tl == 28 and ms > 0.0
    # a different pole range and buffers get their own graphs
    c = [host(t) for t in p.apply_partial(0, 100, *f)]
    d = [host(t) for t in p.apply_partial(100, p.n_poles, *f)]
    assert rel_l2([x + y for x, y in zip(c, d)], a) < 1e-14


@pytest.mark.parametrize("graphs", [True, False])
def test_run_spectral_resident_matches_repeated_apply(R, graphs):
    """NEXT-4: rexi_run keeps the state in Fourier space between steps (Re projection done
    spectrally); it matches repeated physical steps to rounding."""
    D, tau, K = 64, 0.3, 5
    f = inputs.white_noise(D)
    p = R.Plan(D, tau)
    p.set_graphs(graphs)
    t = [dev(x) for x in f]
    p.run(K, *t)
    q = [dev(x) for x in f]
    for _ in range(K):
        q = list(p.apply(*q))
    assert rel_l2([host(x) for x in t], [host(x) for x in q]) < 1e-13
    # energy after K steps (A skew-symmetric): conserved to tolerance
    e0 = sum(float((x ** 2).sum()) for x in f)
    e1 = sum(float((host(x) ** 2).sum()) for x in t)
    assert abs(e1 - e0) / e0 < 1e-11



@pytest.mark.parametrize("mpt,pu,minb", [(4, 1, 4), (4, 1, 5), (4, 1, 6), (4, 2, 3), (4, 2, 4),
                                         (4, 4, 3), (8, 1, 2), (8, 1, 3), (8, 2, 2), (8, 3, 2),
                                         (8, 4, 2), (8, 8, 2), (8, 2, 3), (8, 4, 3), (8, 8, 3),
                                         (16, 2, 2)])
@pytest.mark.parametrize("D", [4, 8, 16, 32, 64])
def test_pfhr_tunings_vs_oracle(R, mpt, pu, minb, D):
    """R2C-pair kernel (real input): every tuning vs the oracle step, grids with every quad type
    (corner, axis, Nyquist, interior) and ragged tiles."""
    tau = 0.9
    f = inputs.white_noise(D)
    p = R.Plan(D, tau, variant="pfhr")
    p.set_tuning(mpt, pu, minb)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    info = p.info
    ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
    assert rel_l2(got, ref) < TOL


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_apply_full_size_sampled_vs_oracle(R, cfg):
    """The bench's launch configuration (default plan: PFHX octet kernel, chunked schedule,
    whole-step graph) at BASELINE's full sizes, element by element against the oracle on
    sampled modes: the spectrum of the GPU's physical output at K must equal the Hermitian part
    of the oracle's dense-LU pole sum, (A(K) + conj A(-K)) / 2 — the spectral form of
    Re(IDFT(.)). Input spectra: the oracle's naive DFT at 512^2, numpy's FFT
    above (the naive O(D^3) DFT takes minutes to hours there); output spectra: numpy's FFT."""
    D, tau, tol, S = {"c2": (512, 1.0, 1e-8, 2048), "c3": (1024, 0.1, 1e-12, 1024),
                      "c4": (4096, 1.0, 1e-12, 256)}[cfg]
    f = inputs.white_noise(D, seed=13)
    p = R.Plan(D, tau, tol=tol)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    ml, mk = inputs.sample_modes(D, S)
    mlm, mkm = (-ml) % D, (-mk) % D
    if D <= 512:
        F = lrsw.spectral_fields(*f)
    else:
        F = np.stack([np.fft.fft2(x) / D ** 2 for x in f], axis=-1)
    Fs, Fm = F[ml, mk, :], F[mlm, mkm, :]
    del F
    got_s = np.stack([(np.fft.fft2(g) / D ** 2)[ml, mk] for g in got], axis=-1)
    n, al, c1, c2, gm = oracle_terms(p).half()
    A = lrsw.rexii_pole_sum(D, tau, Fs, ml, mk, al, c1, c2, gm)
    Am = lrsw.rexii_pole_sum(D, tau, Fm, mlm, mkm, al, c1, c2, gm)
    ref = (A + np.conj(Am)) / 2
    err = float(np.linalg.norm(got_s - ref) / np.linalg.norm(ref))
    assert err < TOL, err


@pytest.mark.parametrize("variant", ["pfhx", "pfhr"])
def test_r2c_c2_full_size_properties(R, variant):
    """The default (PFHX) and the collapsed PFHR at the bench configuration: vs DZ3 (all
    per-pole components formed) and vs the exact propagator."""
    D = 512
    f = inputs.gaussian_scenario(D)
    t = [dev(x) for x in f]
    a = [host(x) for x in R.Plan(D, 1.0, tol=1e-8, variant=variant).apply(*t)]
    b = [host(x) for x in R.Plan(D, 1.0, tol=1e-8, variant="dz3").apply(*t)]
    assert rel_l2(a, b) < TOL
    assert rel_l2(a, lrsw.exact_step(*f, 1.0)) < 1e-8


@pytest.mark.parametrize("pu,minb", [(1, 2), (2, 2), (4, 2), (8, 2), (1, 3), (2, 3), (4, 3), (8, 3)])
@pytest.mark.parametrize("D", [4, 8, 16, 32, 64])
def test_pfhx_tunings_vs_oracle(R, pu, minb, D):
    """Explicit-solve R2C kernel (the default): every tuning vs the oracle step on grids with
    every quad type (corner, axis, Nyquist, interior, half-discarded octets) and ragged tiles."""
    tau = 0.9
    f = inputs.white_noise(D)
    p = R.Plan(D, tau, variant="pfhx")
    p.set_tuning(8, pu, minb)
    p.set_schedule("chunked")   # the multi-launch kernel (AUTO would fuse these small steps)
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    assert p.info["last_schedule"] == 1
    info = p.info
    ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
    assert rel_l2(got, ref) < TOL


def test_h_auto_c2(R):
    """NEXT-2: h chosen from tol (h_for_tol) at the bench configuration: ~3x fewer poles and
    still within tol of the exact propagator; parity with the oracle at a small size."""
    D = 512
    f = inputs.gaussian_scenario(D)
    p = R.Plan(D, 1.0, tol=1e-8, h="auto")
    info = p.info
    assert info["h"] > 1.4 and p.n_poles < 1600
    got = [host(t) for t in p.apply(*(dev(x) for x in f))]
    assert rel_l2(got, lrsw.exact_step(*f, 1.0)) < 1e-8
    D = 32
    g = inputs.white_noise(D)
    q = R.Plan(D, 2.0, tol=1e-8, h="auto")
    got = [host(t) for t in q.apply(*(dev(x) for x in g))]
    ref = lrsw.rexii_step(*g, 2.0, q.info["h"], q.info["M"])
    assert rel_l2(got, ref) < TOL
    assert rel_l2(got, lrsw.exact_step(*g, 2.0)) < 1e-8


def test_refit_table_on_gpu(R):
    """NEXT-2: a plan using the planner's least-squares refit of the Gaussian (instead of
    Appendix A) reaches the same accuracy against the exact propagator; a smaller L (fewer
    terms, N = M + L) works too."""
    D, tau = 64, 1.0
    f = inputs.white_noise(D)
    t = [dev(x) for x in f]
    ex = lrsw.exact_step(*f, tau)
    p = R.Plan(D, tau, tol=1e-12)
    base = [host(x) for x in p.apply(*t)]
    mu, a, defect = R.fit_gaussian(24)
    p.set_table(mu, a)
    got = [host(x) for x in p.apply(*t)]
    assert rel_l2(got, ex) < 1e-12 and rel_l2(base, ex) < 1e-12
    mu20, a20, d20 = R.fit_gaussian(20, mu)
    p.set_table(mu20, a20)
    assert p.n_poles == p.info["M"] + 21
    got20 = [host(x) for x in p.apply(*t)]
    assert rel_l2(got20, ex) < max(1e-10, 100 * d20)


# ----------------------------------------------------------------------------- edge cases
def test_tau_zero_and_negative(R):
    """tau = 0 gives the identity (to the approximation's r(0) error); a step of -tau undoes a
    step of +tau (e^{-tau A} e^{tau A} = I; REXII is valid for both signs, eq:modifiedRexi)."""
    D = 64
    f = inputs.white_noise(D)
    t = [dev(x) for x in f]
    p0 = R.Plan(D, 0.0)
    assert rel_l2([host(x) for x in p0.apply(*t)], f) < 1e-13
    pp, pm = R.Plan(D, 0.7), R.Plan(D, -0.7)
    back = pm.apply(*pp.apply(*t))
    assert rel_l2([host(x) for x in back], f) < 1e-12
    # and -tau matches the oracle too
    ref = lrsw.rexii_step(*f, -0.7, pm.info["h"], pm.info["M"])
    assert rel_l2([host(x) for x in pm.apply(*t)], ref) < TOL


def test_zero_input_and_single_mode(R):
    """Linear map: zero in, zero out; a single Fourier mode stays a single mode (per-mode solves,
    PAPER.md:497), matching the exact propagator."""
    D = 32
    p = R.Plan(D, 1.0)
    z = [dev(np.zeros((D, D))) for _ in range(3)]
    assert max(float(x.abs().max()) for x in p.apply(*z)) == 0.0
    X, Y = inputs.grid(D)
    f = (np.sin(6 * np.pi * X) * np.cos(4 * np.pi * Y), np.zeros((D, D)), np.zeros((D, D)))
    got = [host(x) for x in p.apply(*(dev(x) for x in f))]
    assert rel_l2(got, lrsw.exact_step(*f, 1.0)) < 1e-12
    Fg = np.fft.fft2(got[0])
    Fg[np.abs(Fg) < 1e-9 * np.abs(Fg).max()] = 0
    assert set(zip(*np.nonzero(Fg))) <= {(l % D, k % D) for l in (2, -2) for k in (3, -3)}


def test_max_grid_8192_small_tau(R):
    """Largest supported grid (D = 8192, 67M modes, 3.2 GB per spectral array): a short step
    conserves energy and the mean of eta; the forward FFT matches the DFT on sampled entries."""
    import torch
    D = 8192
    p = R.Plan(D, 0.002, tol=1e-10)
    g = np.random.Generator(np.random.PCG64(4))
    X = g.standard_normal((D, D))
    t = [torch.from_numpy(X).cuda(), torch.zeros((D, D), dtype=torch.float64, device="cuda"),
         torch.zeros((D, D), dtype=torch.float64, device="cuda")]
    F0 = host(p.forward(*t)[0])
    x = np.arange(D)
    for (l, k) in [(0, 0), (1, 4095), (4096, 4096), (8191, 3)]:
        ph = np.exp(-2j * np.pi * ((k * x[None, :] + l * x[:, None]) % D) / D)
        assert abs(F0[l, k] - (X * ph).sum() / D ** 2) < 1e-15
    out = p.apply(*t)
    e0 = float((t[0] ** 2).sum())
    e1 = sum(float((o ** 2).sum()) for o in out)
    assert abs(e1 - e0) / e0 < 1e-10
    assert abs(float(out[0].mean()) - float(t[0].mean())) < 1e-13
