"""Stage clock marks of the fused DSMEM step (REXI_SMALL_TRACE=1, graphs off): per CTA, clock64
deltas from kernel entry at marks 1..12 (preload, A fft, A stores, B, C setup, C tile, C part,
C sync, D, hand-off, E, F), medians over steps, after an L2 flush before every step.
    REXI_SMALL_TRACE=1 python tools/trace_c1.py [D tau] 2> trace.log"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

D = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
p = rexi.Plan(D, tau, tol=1e-12)
p.set_graphs(False)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(20):
    flush.zero_()
    p.apply(*f)
torch.cuda.synchronize()
