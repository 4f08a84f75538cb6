"""(Test-side script: it uses the oracle's exact propagator.) Print the CUDA path's one-step max-norm errors for the paper's Table 2-7 rows (GPU box)."""
import json
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import torch

from conftest import read_paper_tables
from oracle import lrsw
from paper_2008_11607_b200 import inputs, rexi
from test_gpu_parity import EXTRA_ROWS, _SCEN

D = 128
for row in read_paper_tables() + EXTRA_ROWS:
    f = _SCEN[row["scenario"]](D)
    p = rexi.Plan(D, row["tau"], h=row["h"], M=row["M"], method=row["method"].lower())
    t = [torch.from_numpy(x).cuda() for x in f]
    p.apply(*t)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = p.apply(*t)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    got = [o.cpu().numpy() for o in out]
    ex = lrsw.exact_step(*f, row["tau"])
    err = max(float(np.abs(a - b).max()) for a, b in zip(got, ex))
    print(json.dumps({**row, "gpu_err": err, "gpu_ms": dt * 1e3, "n_poles": p.n_poles}), flush=True)
