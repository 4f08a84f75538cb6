"""Writes the PFHX results of a few configurations to an .npz (argv[1]): run once with the default
bulk-copy pole-table staging and once with REXI_R2X_BULK=0 (register-staged copy); the two
kernels differ only in how the pole table reaches shared memory, so the results must be
bit-identical (tests/test_gpu_staging.py)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2008_11607_b200 import inputs, rexi  # noqa: E402

res = {}
for D, tau, tol, b, e in ((64, 1.0, 1e-12, 0, None), (512, 1.0, 1e-8, 0, None), (512, 1.0, 1e-8, 100, 1337),
                          (1024, 0.1, 1e-12, 0, None), (128, 3.0, 1e-12, 5, 6)):
    p = rexi.Plan(D, tau, tol=tol)
    p.set_schedule("chunked")   # the pole kernel also where AUTO would fuse the small steps
    f = [torch.from_numpy(x).cuda() for x in inputs.white_noise(D, seed=D + 7)]
    e = p.n_poles if e is None else e
    out = p.apply_partial(b, e, *f)
    res[f"D{D}_b{b}_e{e}"] = np.stack([o.cpu().numpy() for o in out])
    if b == 0 and e == p.n_poles:
        res[f"D{D}_apply"] = np.stack([o.cpu().numpy() for o in p.apply(*f)])
np.savez(sys.argv[1], **res)
print("ok", len(res))
