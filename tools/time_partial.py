"""One rank's share of a pole-parallel step, measured on one GPU: rexi_apply_partial over the
first 1/P of the poles (P = 1, 2, 4, 8), L2 flushed before every step, CUDA events on the
launching stream, median — the per-rank compute of bench.py --gpus P without the all-reduce
(the S4 transfer is not measurable on a one-GPU box).

    python tools/time_partial.py [c2|c3|c4] [steps]
"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi
from paper_2008_11607_b200.distributed import pole_partition

CFG = {"c2": (512, 1.0, 1e-8), "c3": (1024, 0.1, 1e-12), "c4": (4096, 1.0, 1e-12)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
D, tau, tol = CFG[name]
plan = rexi.Plan(D, tau, tol=tol)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
out = torch.empty((3, D, D), dtype=torch.float64, device="cuda")
o3 = (out[0], out[1], out[2])
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
n = plan.n_poles
for P in (1, 2, 4, 8):
    b, e = pole_partition(n, P, 0)
    for _ in range(5):
        plan.apply_partial(b, e, *f, out=o3)
    plan.timing_enable(True)
    plan.timing_read()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        plan.apply_partial(b, e, *f, out=o3)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(c) for a, c in ev)
    k = plan.timing_read()
    plan.timing_enable(False)
    print(json.dumps({"config": name, "P": P, "poles": [b, e], "partial_ms": ms,
                      "pole_kernel_ms": k[0] / max(1, k[1]), "non_pole_ms": ms - k[0] / max(1, k[1])}), flush=True)
