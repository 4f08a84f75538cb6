"""(Test-side script: it uses the oracle's exact propagator.) C5 sweep (BASELINE configs[4]): error vs the exact propagator and
throughput vs the number of REXII terms, on the GPU path (GPU box).

    python tests/scripts/sweep.py [D] > profiles/r01_sweep_c5_<D>.jsonl

White-noise fields (every Fourier mode excited, so the largest |K| of the grid — the rho of
the M rule — is present; the Gaussian bump's spectrum dies long before it and hides the
truncation cliff), one step per (tau, h, M), M = the paper's rule for tol 1e-12
(rexi_rule_M) plus an offset; error = relative L2 over (eta, u, v) and max-norm vs
lrsw.exact_step (per-mode closed-form exponential); time = CUDA events around the pole kernel
and around the whole step (whole-step graph), median of 5 after warm-up."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import lrsw
from paper_2008_11607_b200 import inputs, rexi

D = int(sys.argv[1]) if len(sys.argv) > 1 else 512
f = inputs.white_noise(D, seed=17)
fd = [torch.from_numpy(x).cuda() for x in f]
for tau in (0.01, 0.1, 1.0, 10.0, 50.0):
    ex = lrsw.exact_step(*f, tau)
    nex = np.sqrt(sum(float((x ** 2).sum()) for x in ex))
    for h in (0.3, 0.5, 1.0):
        M0 = rexi.rule_M(D, tau, 1e-12, h)
        for dM in (-12, -8, -4, -2, 0, 4):
            M = M0 + dM
            if M < 12:
                continue
            p = rexi.Plan(D, tau, h=h, M=M)
            out = p.apply(*fd)
            torch.cuda.synchronize()
            got = [o.cpu().numpy() for o in out]
            rel = np.sqrt(sum(float(((a - b) ** 2).sum()) for a, b in zip(got, ex))) / nex
            mx = max(float(np.abs(a - b).max()) for a, b in zip(got, ex))
            reps = 5
            step_ms, pole_ms = [], []
            for _ in range(reps):
                p.timing_enable(True)
                p.timing_read()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                p.apply(*fd, out=out)
                e1.record()
                torch.cuda.synchronize()
                ms, n, _ = p.timing_read()
                p.timing_enable(False)
                step_ms.append(e0.elapsed_time(e1))
                pole_ms.append(ms / max(1, n))
            st, pk = float(np.median(step_ms)), float(np.median(pole_ms))
            npl = p.n_poles
            print(json.dumps({"D": D, "tau": tau, "h": h, "M": M, "M_rule_1e-12": M0, "dM": dM,
                              "n_poles": npl, "rel_l2_vs_exact": rel, "max_err_vs_exact": mx,
                              "step_ms": st, "pole_kernel_ms": pk, "steps_per_s": 1e3 / st,
                              "pole_gp_per_s": npl * D * D / (st / 1e3)}), flush=True)
