"""The default PFHX kernel streams the pole table into shared memory by bulk copies on the TMA
engine (cp.async.bulk + mbarrier, double-buffered: pole_kernel_r2x_bulk); REXI_R2X_BULK=0 selects
the register-staged copy (pole_kernel_r2x). Same arithmetic in the same order, so the results
must be bit-identical: a missed or early mbarrier wait, a refilled buffer still being read, or a
wrong tile offset would change them (full grids, a ragged pole range, a one-pole range, several
tiles per chunk)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bulk_staging_bit_identical_to_register_staging(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2008_11607_b200 import build
    build.build()
    script = os.path.join(ROOT, "tests", "scripts", "staging_identity.py")
    outs = {}
    for mode in ("1", "0"):
        path = str(tmp_path / f"r{mode}.npz")
        env = dict(os.environ, REXI_R2X_BULK=mode)
        r = subprocess.run([sys.executable, script, path], env=env, capture_output=True, text=True,
                           timeout=600, cwd=ROOT)
        assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
        outs[mode] = np.load(path)
    assert sorted(outs["1"].files) == sorted(outs["0"].files) and len(outs["1"].files) == 8
    for k in outs["1"].files:
        a, b = outs["1"][k], outs["0"][k]
        assert np.all(np.isfinite(a)), k
        assert np.array_equal(a, b), (k, float(np.abs(a - b).max()))
