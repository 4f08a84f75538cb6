"""Time the non-pole stages (forward FFT, inverse FFT, poles call) with CUDA events (GPU box)."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

for D, tau in ((64, 0.02), (512, 1.0), (1024, 0.1), (4096, 1.0)):
    p = rexi.Plan(D, tau, tol=1e-8)
    f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
    F = p.forward(*f)
    out = p.inverse(F)
    reps = 50 if D < 4096 else 5
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    for _ in range(reps):
        p.forward(*f, fhat=F)
    e[1].record()
    for _ in range(reps):
        p.inverse(F, out=out)
    e[2].record()
    acc = torch.empty_like(F)
    for _ in range(reps if D < 4096 else 1):
        p.poles(F, 0, 1, acc=acc)
    e[3].record()
    torch.cuda.synchronize()
    fw = e[0].elapsed_time(e[1]) / reps * 1e3
    iv = e[1].elapsed_time(e[2]) / reps * 1e3
    po = e[2].elapsed_time(e[3]) / (reps if D < 4096 else 1) * 1e3
    gb = 3 * D * D * (8 + 16 + 16 + 16) / 1e9   # row r2c + col c2c bytes
    print(json.dumps({"D": D, "forward_us": fw, "inverse_us": iv, "poles_1pole_us": po,
                      "forward_GBps": gb / (fw * 1e-6)}), flush=True)
