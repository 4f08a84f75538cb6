"""Example: the paper's Gaussian-bump scenario (eq:GAUSSIANSCENARIO) stepped with REXII on a B200.

    python examples/lrsw_gaussian.py [D] [tau] [steps]

Creates a plan (term count from the paper's rule for tol 1e-12), runs `steps` steps in place
with rexi_run (state kept in Fourier space between steps), and prints the energy drift (A is
real skew-symmetric, so e^{tA} conserves eta^2 + u^2 + v^2) and the mean of eta. Accuracy
against the exact propagator is what tests/ checks (the oracle is test infrastructure)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2008_11607_b200 import inputs, rexi  # noqa: E402

D = int(sys.argv[1]) if len(sys.argv) > 1 else 512
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10

f0 = inputs.gaussian_scenario(D)
plan = rexi.Plan(D, tau, tol=1e-12)
info = plan.info
print(f"D={D} tau={tau} h={info['h']} M={info['M']} poles={info['n_poles']} "
      f"predicted floor={info['predicted_floor']:.1e}")
state = [torch.from_numpy(x.copy()).cuda() for x in f0]
torch.cuda.synchronize()
t0 = time.perf_counter()
plan.run(steps, *state)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{steps} steps in {dt * 1e3:.1f} ms ({dt / steps * 1e3:.2f} ms/step, "
      f"{info['n_poles'] * D * D * steps / dt:.3g} pole-gridpoint solves/s)")

got = [x.cpu().numpy() for x in state]
e0 = sum((x ** 2).sum() for x in f0)
e1 = sum((x ** 2).sum() for x in got)
print(f"after T = {tau * steps}: energy drift {abs(e1 - e0) / e0:.2e}, "
      f"mean(eta) {got[0].mean():.6e} (initial {f0[0].mean():.6e})")
