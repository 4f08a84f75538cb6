"""A/B the pole-kernel schedules (chunked vs stream-K) on one config, interleaved (GPU box).
    python tools/ab_sched.py c2 [rounds] [pu list, e.g. 1,2,8]"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pus = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2]
D, tau, tol = {"c2": (512, 1.0, 1e-8), "c3": (1024, 0.1, 1e-12), "c4": (4096, 1.0, 1e-12)}[cfg]
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
plans = {}
for sched in ("chunked", "streamk"):
    for pu in pus:
        p = rexi.Plan(D, tau, tol=tol)
        p.set_schedule(sched)
        p.set_tuning(8, pu, 2)
        out = p.apply(*f)
        plans[(sched, pu)] = (p, out)
torch.cuda.synchronize()
reps = 20 if D <= 1024 else 1
res = {k: [] for k in plans}
for _ in range(rounds):
    for k, (p, out) in plans.items():
        p.timing_enable(True)
        p.timing_read()
        for _ in range(reps):
            p.apply(*f, out=out)
        ms, n, _ = p.timing_read()
        p.timing_enable(False)
        res[k].append(ms / n)
for k, v in res.items():
    print(cfg, k, "pole kernel ms", " ".join(f"{x:.4f}" for x in v), "last_schedule", plans[k][0].info["last_schedule"])
