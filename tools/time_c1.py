"""Time the C1 step (fused small-grid kernel) with CUDA events: python tools/time_c1.py [D tau]"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

D = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
p = rexi.Plan(D, tau, tol=1e-12)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
out = p.apply(*f)
p.timing_enable(True)
for _ in range(20):
    p.apply(*f, out=out)
torch.cuda.synchronize()
p.timing_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    p.apply(*f, out=out)
e1.record()
torch.cuda.synchronize()
ms, pl, tl = p.timing_read()
print(f"D={D} step {e0.elapsed_time(e1) / 200 * 1e3:.1f} us, kernel {ms / pl * 1e3:.1f} us ({pl} launches)")
