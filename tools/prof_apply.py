"""Run a few rexi_apply steps of a config (for ncu captures of the non-pole kernels on the
apply path: forward FFT, finish, K = 0 fix-up, inverse FFT of the Hermitian accumulator).
    python tools/prof_apply.py <config> [steps]"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

cfg = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
D, tau, tol = {"c1": (64, 0.02, 1e-12), "c2": (512, 1.0, 1e-8), "c3": (1024, 0.1, 1e-12),
               "c4": (4096, 1.0, 1e-12)}[cfg]
p = rexi.Plan(D, tau, tol=tol)
p.set_graphs(False)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
for _ in range(steps):
    out = p.apply(*f)
torch.cuda.synchronize()
print("ok")
