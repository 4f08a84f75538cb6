"""Pole-kernel time over pole counts at 512^2 (chunked schedule): per-pole slope and per-launch
intercept of the PFHX kernel, from small ranges (one wave or less) to the full C2 range.
    python tools/time_pole_counts.py [counts...]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2008_11607_b200 import inputs, rexi  # noqa: E402

D = 512
plan = rexi.Plan(D, 1.0, tol=1e-8)
plan.set_schedule("chunked")
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
out = torch.empty((3, D, D), dtype=torch.float64, device="cuda")
o3 = (out[0], out[1], out[2])
counts = [int(x) for x in sys.argv[1:]] or [8, 16, 32, 64, 128, 256, 572, 1144, 2291, 4583]
for e in counts:
    for _ in range(3):
        plan.apply_partial(0, e, *f, out=o3)
    plan.timing_enable(True)
    plan.timing_read()
    torch.cuda.synchronize()
    for _ in range(100):
        plan.apply_partial(0, e, *f, out=o3)
    torch.cuda.synchronize()
    k = plan.timing_read()
    plan.timing_enable(False)
    ms = k[0] / k[1]
    print(f"poles {e}: pole kernel {ms * 1e3:.2f} us, {ms * 1e3 / e:.4f} us/pole", flush=True)
