"""Workload for the bounds-checked library (librexi_checked.so, REXI_CHECKED): the replacement
for compute-sanitizer memcheck/racecheck, which this GPU pool does not allow.

Run with REXI_LIB pointing at librexi_checked.so (tests/test_gpu_checked.py does): every kernel
of the default and alternative paths runs with device-side bounds asserts on its global and
shared-memory indices (a failed assert traps: the process then fails), NaN-poisoned workspace and
shared memory (a read of an unwritten slot reaches the output), and each result is
  * compared with the oracle (a NaN or a wrong value fails), and
  * recomputed and compared BIT FOR BIT (a shared-memory or inter-CTA race would show as
    run-to-run differences).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from oracle import lrsw
from paper_2008_11607_b200 import inputs, rexi

assert os.path.basename(rexi.LIB_PATH) == "librexi_checked.so", rexi.LIB_PATH


def rel(a, b):
    a = np.concatenate([np.ravel(x) for x in a])
    b = np.concatenate([np.ravel(x) for x in b])
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def host(ts):
    return [t.cpu().numpy() for t in ts]


def check(name, fn, ref, tol=1e-12):
    a = host(fn())
    b = host(fn())
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        if not np.array_equal(x, y):
            raise SystemExit(f"{name}: run-to-run difference (race?)")
    if not all(np.isfinite(x).all() for x in a):
        raise SystemExit(f"{name}: non-finite output (read of an unwritten slot?)")
    e = rel(a, ref)
    if not e < tol:
        raise SystemExit(f"{name}: rel err {e:.3e} vs oracle")
    print(f"{name}: ok ({e:.2e})", flush=True)


cases = [(4, 0.5, 1e-12), (8, 0.7, 1e-12), (16, 1.0, 1e-12), (64, 0.02, 1e-12), (64, 1.0, 1e-12),
         (128, 0.3, 1e-12)]
for D, tau, tol in cases:
    f = inputs.white_noise(D, seed=91)
    fd = [torch.from_numpy(x).cuda() for x in f]
    for variant, sched in (("pfhx", "chunked"), ("pfhx", "fused"), ("pfhr", "chunked"),
                           ("pfhr", "streamk"), ("pfh", "auto"), ("dz", "auto"), ("uv", "auto")):
        p = rexi.Plan(D, tau, tol=tol, variant=variant)
        p.set_schedule(sched)
        info = p.info
        ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
        check(f"D={D} tau={tau} {variant}/{sched} apply", lambda: p.apply(*fd), ref)
        b, e = 0, max(1, p.n_poles // 3)
        from oracle import coeffs as C
        n, al, c1, c2, g = C.rexii_terms(info["h"], info["M"]).half()
        F = lrsw.spectral_fields(*f)
        ml, mk = lrsw.all_modes(D)
        acc = lrsw.rexii_pole_sum(D, tau, F[ml, mk], ml, mk, al[b:e], c1[b:e], c2[b:e], g[b:e])
        A = np.zeros((D, D, 3), complex)
        A[ml, mk] = acc
        refp = [lrsw.idft2_real(A[..., c]) for c in range(3)]
        check(f"D={D} tau={tau} {variant}/{sched} apply_partial", lambda: p.apply_partial(b, e, *fd), refp)
    # spectral-resident steps, host buffers, the Hermitian mirror
    p = rexi.Plan(D, tau, tol=tol)
    info = p.info
    g3 = f
    for _ in range(2):
        g3 = lrsw.rexii_step(*g3, tau, info["h"], info["M"])

    def run2():
        x = [t.clone() for t in fd]
        p.run(2, *x)
        return x
    check(f"D={D} tau={tau} run(2)", run2, g3)
    ref = lrsw.rexii_step(*f, tau, info["h"], info["M"])
    check(f"D={D} tau={tau} apply_host", lambda: [torch.from_numpy(o) for o in
                                                  p.apply_host(*[np.ascontiguousarray(x) for x in f])], ref)
# large grids: the radix-16 row passes and the cluster column passes (2048^2, 4096^2) of the
# apply path and of rexi_forward / rexi_inverse — asserts, NaN-poisoned workspace, bit-for-bit
# repeat, and the transform round trip inverse(forward(x)) = x (a property at any size; the
# values themselves are checked against the oracle by the regular GPU tests on sampled modes)
for D in (1024, 2048, 4096):
    f = inputs.white_noise(D, seed=93)
    fd = [torch.from_numpy(x).cuda() for x in f]
    tau = 1e-5
    p = rexi.Plan(D, tau, tol=1e-8)
    p.set_schedule("chunked")
    a1 = host(p.apply(*fd))
    a2 = host(p.apply(*fd))
    for x, y in zip(a1, a2):
        if not np.array_equal(x, y):
            raise SystemExit(f"D={D} apply: run-to-run difference (race?)")
    if not all(np.isfinite(x).all() for x in a1):
        raise SystemExit(f"D={D} apply: non-finite output (read of an unwritten slot?)")
    # A is skew-symmetric with spectral radius rho = sqrt(2) pi D (eq:lswRoh), so
    # ||e^{tau A} f - f|| <= tau rho ||f|| (+ the REXII tolerance)
    e_id, bound = rel(a1, f), 1.01 * tau * np.sqrt(2.0) * np.pi * D + 1e-7
    if not e_id < bound:
        raise SystemExit(f"D={D} apply: {e_id:.3e} from the input, bound {bound:.3e}")
    F = p.forward(*fd)
    back = host(p.inverse(F))
    e_rt = rel(back, f)
    if not e_rt < 1e-13:
        raise SystemExit(f"D={D} round trip {e_rt:.3e}")
    print(f"D={D} apply (chunked, cluster column passes from 2048) + round trip: ok ({e_rt:.2e})", flush=True)
print("CHECKED OK")
