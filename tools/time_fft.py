"""Time the forward and inverse real 2-D FFT of a plan (GPU box): python tools/time_fft.py D"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

D = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = rexi.Plan(D, 0.1, tol=1e-8)
p.set_graphs(False)
f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D)]
F = p.forward(*f)
o = p.inverse(F)
torch.cuda.synchronize()
for name, fn in (("forward", lambda: p.forward(*f, fhat=F)), ("inverse", lambda: p.inverse(F, out=o))):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(D, name, f"{e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
