"""Bit-for-bit repeatability of apply / forward / inverse at a large grid (race hunt):
    python tools/race_probe.py D [reps]"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2008_11607_b200 import inputs, rexi

D = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D, seed=93)]
p = rexi.Plan(D, 1e-5, tol=1e-8)
p.set_schedule("chunked")


def diff(name, fn):
    a = [t.clone() for t in fn()]
    worst = 0
    for _ in range(reps):
        b = fn()
        for x, y in zip(a, b):
            nd = int((x != y).sum().item())
            if nd:
                idx = torch.nonzero(x != y)[:3].tolist()
                print(f"  {name}: {nd} entries differ, e.g. {idx}, max |diff| {float((x - y).abs().max()):.3e}")
            worst = max(worst, nd)
    print(f"{name}: {'bit-for-bit' if worst == 0 else 'DIFFERS'}", flush=True)


Z = torch.zeros((D, D), dtype=torch.float64, device="cuda")
diff("forward (full spectrum)", lambda: p.forward(*f))
F = p.forward(*f)
diff("inverse (symmetrising)", lambda: p.inverse(F))
diff("apply", lambda: p.apply(*f))
