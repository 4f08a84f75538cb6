"""Run the pole kernel a few times with a given tuning (for ncu captures on the GPU box).
    python tools/prof_pole.py <config> <variant> <mpt> <pu> <minb>"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

cfg, variant, mpt, pu, minb = sys.argv[1], sys.argv[2], *map(int, sys.argv[3:6])
D, tau, tol = {"c1": (64, 0.02, 1e-12), "c2": (512, 1.0, 1e-8), "c3": (1024, 0.1, 1e-12),
               "c4": (4096, 1.0, 1e-12)}[cfg]
p = rexi.Plan(D, tau, tol=tol, variant=variant)
p.set_tuning(mpt, pu, minb)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
F = p.forward(*f)
acc = p.poles(F)
for _ in range(3):
    p.poles(F, acc=acc)
torch.cuda.synchronize()
print("ok")
