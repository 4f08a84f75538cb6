"""Per-step time of rexi_run (spectral-resident multi-step) at a small grid: the fused one-launch
run (AUTO) against the chunked spectral path (set_schedule('chunked')), CUDA events, no L2 flush
between steps of a run (they are one call):  python tools/time_run.py [D tau K]"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

D = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
K = int(sys.argv[3]) if len(sys.argv) > 3 else 100
f0 = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for sched in ("auto", "chunked"):
    p = rexi.Plan(D, tau, tol=1e-12)
    p.set_schedule(sched)
    ts = []
    for rep in range(12):
        f = [t.clone() for t in f0]
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.run(K, *f)
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3 / K)
    print(f"D={D} tau={tau} K={K} {sched}: {statistics.median(ts):.2f} us per step "
          f"(last schedule {p.info['last_schedule']})", flush=True)
