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
print("CHECKED OK")
