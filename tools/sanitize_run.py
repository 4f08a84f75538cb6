"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck) through the C ABI:
C1 (64^2, tau 0.02) and a small 512^2 step (tau 0.02, ~120 poles) with the default PFHX kernel,
the PFHR and generic kernels, rexi_apply_partial, rexi_run and the host-buffer path — i.e. the
R2C pole kernels, the four FFT passes, finish, the K = 0 fix-up and the Hermitian projection.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2008_11607_b200 import inputs, rexi

for D, tau, tol in ((64, 0.02, 1e-12), (512, 0.02, 1e-8)):
    f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D)]
    for variant in ("pfhx", "pfhr", "pfh"):
        p = rexi.Plan(D, tau, tol=tol, variant=variant)
        out = p.apply(*f)
        n = p.n_poles
        p.apply_partial(0, n // 3, *f)
        torch.cuda.synchronize()
        print(f"D={D} {variant}: poles={n} |eta'|={float(out[0].norm()):.6e}", flush=True)
    p = rexi.Plan(D, tau, tol=tol)
    g = [x.clone() for x in f]
    p.run(2, *g)
    h = [np.ascontiguousarray(x.cpu().numpy()) for x in f]
    p.apply_host(*[torch.from_numpy(x) for x in h])
    torch.cuda.synchronize()
print("sanitize workload done")
