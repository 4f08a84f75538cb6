"""The bounds-checked library (REXI_CHECKED) on every kernel path, in a subprocess: device asserts
on all global / shared-memory indices, NaN-poisoned workspace and shared memory, results vs the
oracle and bit-for-bit repeatable (tests/scripts/checked_run.py). Stands in for compute-sanitizer
memcheck / racecheck, which this GPU pool does not run."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_library_all_paths():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2008_11607_b200 import build
    lib = build.build_checked()
    env = dict(os.environ, REXI_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "scripts", "checked_run.py")], env=env,
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    with open(os.path.join(ROOT, "gpurun_out", "checked_run.log") if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
              else os.devnull, "w") as fh:
        fh.write(out)
    assert "REXI_CHECKED:" not in out, out[-4000:]
    assert r.returncode == 0 and "CHECKED OK" in out, out[-4000:]
