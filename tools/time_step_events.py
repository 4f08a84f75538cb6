"""Per-step CUDA-event times of one config the way bench.py takes them (L2 flush before every
step, events on the launching stream, median), with the library's pole-kernel timing events
on and off; flush=2: a busy-wait kernel instead of the flush (warm L2, host ahead of the GPU);
flush=0: back to back (host-bound for small steps).

    python tools/time_step_events.py [c1|c2|c3] [steps]
"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2008_11607_b200 import inputs, rexi

CFG = {"c1": (64, 0.02, 1e-12), "c2": (512, 1.0, 1e-8), "c3": (1024, 0.1, 1e-12)}
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
D, tau, tol = CFG[name]
plan = rexi.Plan(D, tau, tol=tol)
f = [torch.from_numpy(x).cuda() for x in inputs.gaussian_scenario(D)]
out = torch.empty((3, D, D), dtype=torch.float64, device="cuda")
o3 = (out[0], out[1], out[2])
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
for _ in range(20):
    plan.apply(*f, out=o3)
torch.cuda.synchronize()


def run(timing, do_flush):
    plan.timing_enable(timing)
    plan.timing_read()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for _ in range(5):
        plan.apply(*f, out=o3)
    torch.cuda.synchronize()
    for i in range(steps):
        if do_flush == 1:
            flush.zero_()
        elif do_flush == 2:
            torch.cuda._sleep(100000)   # ~50 us busy wait: the host runs ahead, L2 stays warm
        ev[i][0].record(stream)
        plan.apply(*f, out=o3)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    k = plan.timing_read() if timing else (0.0, 0, 0)
    plan.timing_enable(False)
    kern = k[0] / k[1] * 1e3 if timing and k[1] else float("nan")
    return statistics.median(ms) * 1e3, kern, statistics.mean(ms) * 1e3


for timing in (False, True):
    for do_flush in (1, 2, 0):
        med, kern, mean = run(timing, do_flush)
        print(f"{name} D={D}: timing={int(timing)} flush={int(do_flush)} step median {med:.2f} us (mean {mean:.2f})"
              + (f", pole/fused kernel {kern:.2f} us" if timing else ""))
