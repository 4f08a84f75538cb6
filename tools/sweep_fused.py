"""Step time of the chunked multi-launch path against the fused step with 1..8 clusters, for small
grids and growing pole counts (L2 flushed before every step, CUDA events, median and mean):
the measurements behind AUTO's fused / chunked choice and the automatic cluster count.
    python tools/sweep_fused.py > sweep_fused.jsonl"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()


def time_steps(plan, f, out, steps=150):
    for _ in range(10):
        plan.apply(*f, out=out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        plan.apply(*f, out=out)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in ev]
    return statistics.median(ms), statistics.mean(ms)


cases = [(64, 0.02), (64, 0.1), (64, 0.3), (64, 1.0), (32, 1.0), (128, 0.02), (128, 0.1), (128, 0.3)]
for D, tau in cases:
    f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
    o = torch.empty((3, D, D), dtype=torch.float64, device="cuda")
    out = (o[0], o[1], o[2])
    p = rexi.Plan(D, tau, tol=1e-12)
    n = p.info["n_poles"]
    p.set_schedule("chunked")
    row = {"D": D, "tau": tau, "poles": n, "chunked_us": time_steps(p, f, out)}
    p.set_schedule("fused")
    for nc in (1, 2, 3, 4, 6, 8):
        if nc > n:
            continue
        p.set_fused_clusters(nc)
        row[f"fused_nc{nc}_us"] = time_steps(p, f, out)
    print(json.dumps(row), flush=True)
