"""Forward transform and whole apply of a tiny-tau plan (a handful of poles, so the FFT passes,
finish and launches dominate) at D: python tools/time_fft_apply.py D"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2008_11607_b200 import inputs, rexi  # noqa: E402

D = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = rexi.Plan(D, 1e-5, tol=1e-8)
p.set_schedule("chunked")
f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D)]
F = p.forward(*f)
out = torch.empty((3, D, D), dtype=torch.float64, device="cuda")
o3 = (out[0], out[1], out[2])
for name, fn in (("forward", lambda: p.forward(*f, fhat=F)), ("apply", lambda: p.apply(*f, out=o3))):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(D, name, f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us (poles {p.n_poles})", flush=True)
