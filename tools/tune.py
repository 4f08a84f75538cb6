"""Time the pole kernel for each (variant, modes-per-thread) on a config (GPU box)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2008_11607_b200 import inputs, rexi

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
D, tau, tol = {"c1": (64, 0.02, 1e-12), "c2": (512, 1.0, 1e-8), "c3": (1024, 0.1, 1e-12),
               "c4": (4096, 1.0, 1e-12)}[cfg]
import os
f = [torch.from_numpy(x).cuda() for x in (inputs.white_noise(D) if os.environ.get("TUNE_INPUT") == "white" else inputs.gaussian_scenario(D))]
res = []
TUNINGS = {"dz": [(1, 1, 8), (2, 1, 4), (2, 1, 5), (3, 1, 4), (4, 1, 3), (4, 1, 4)],
           "uv": [(1, 1, 6), (2, 1, 3), (2, 1, 4), (3, 1, 3), (4, 1, 2), (4, 1, 3)],
           "dz3": [(1, 1, 8), (2, 1, 4), (3, 1, 4), (4, 1, 2), (4, 1, 4)],
           "pf": [(1, 1, 8), (2, 1, 3), (2, 1, 4), (3, 1, 4), (4, 1, 3), (4, 1, 4)],
           "pfh": [(1, 1, 8), (2, 1, 3), (2, 1, 4), (3, 1, 4), (4, 1, 3), (4, 1, 4), (1, 2, 6),
                   (2, 2, 3), (2, 2, 4), (4, 2, 2)],
           "pfhr": [(4, 1, 4), (4, 1, 5), (4, 1, 6), (4, 2, 3), (4, 2, 4), (4, 4, 3), (8, 1, 2),
                    (8, 1, 3), (8, 2, 2), (8, 3, 2), (8, 4, 2), (8, 8, 2), (8, 2, 3), (8, 4, 3), (8, 8, 3), (16, 2, 2)],
           "pfhx": [(8, 1, 2), (8, 2, 2), (8, 4, 2), (8, 8, 2), (8, 1, 3), (8, 2, 3), (8, 4, 3), (8, 8, 3),
                    (8, 4, 5), (8, 8, 5), (8, 4, 6), (8, 8, 6)]}
for variant in sys.argv[2].split(",") if len(sys.argv) > 2 else ("dz", "uv", "dz3", "pf", "pfh", "pfhr"):
    for mpt, pu, minb in TUNINGS[variant]:
        p = rexi.Plan(D, tau, tol=tol, variant=variant)
        p.set_tuning(mpt, pu, minb)
        if os.environ.get("TUNE_SCHEDULE"):
            p.set_schedule(os.environ["TUNE_SCHEDULE"])
        if os.environ.get("TUNE_NOGRAPH"):
            p.set_graphs(False)
        F = p.forward(*f)
        out = p.apply(*f)
        acc = p.poles(F)
        torch.cuda.synchronize()
        p.timing_enable(True)
        p.timing_read()
        reps = 20 if D <= 1024 else 2
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(reps):
            if variant in ("pfhr", "pfhx"):   # the R2C kernels run on the real-input (apply) path
                p.apply(*f, out=out)
            else:
                p.poles(F, acc=acc)
        ev1.record()
        torch.cuda.synchronize()
        ms, pl, tl = p.timing_read()
        info = p.info
        units = info["n_poles"] * D * D
        k_ms = ms / pl
        res.append({"variant": variant, "mpt": mpt, "pu": pu, "minb": minb, "pole_kernel_ms": k_ms,
                    "poles_call_ms": ev0.elapsed_time(ev1) / reps,
                    "pgp_per_s": units / (k_ms / 1e3),
                    "fp64_pipe_frac": info["fp64_ops_per_pole_mode"] * units / (k_ms / 1e3) / (148 * 64 * 1.965e9)})
        print(json.dumps(res[-1]), flush=True)
