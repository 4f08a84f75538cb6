"""Pole-kernel time per pole over pole counts around one rank's share of C2 at P = 8 (chunk lengths
with and without a remainder below the 8-pole loop trip). python tools/time_pole_counts.py"""
import statistics, sys
sys.path.insert(0, ".")
import torch
from paper_2008_11607_b200 import inputs, rexi
D = 512
plan = rexi.Plan(D, 1.0, tol=1e-8)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
out = torch.empty((3, D, D), dtype=torch.float64, device="cuda")
o3 = (out[0], out[1], out[2])
for e in (560, 564, 568, 572, 576, 580, 584, 1144, 1152, 4576, 4583):
    for _ in range(3): plan.apply_partial(0, e, *f, out=o3)
    plan.timing_enable(True); plan.timing_read(); torch.cuda.synchronize()
    for _ in range(100): plan.apply_partial(0, e, *f, out=o3)
    torch.cuda.synchronize()
    k = plan.timing_read(); plan.timing_enable(False)
    ms = k[0] / k[1]
    print(f"poles {e}: pole kernel {ms*1e3:.2f} us, {ms*1e3/e:.4f} us/pole")
