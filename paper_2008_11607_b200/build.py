"""Build librexi.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

    python -m paper_2008_11607_b200.build [--force]
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librexi.so")
# bounds-checked variant (REXI_CHECKED: device asserts on every index of the default path, NaN-
# poisoned workspace and shared memory); loaded only through REXI_LIB by the checked tests
LIB_CHECKED = os.path.join(HERE, "librexi_checked.so")
SOURCES = ["planner.cpp", "fit.cpp", "kernels.cu", "capi.cu", "scalar.cu", "diag.cu"]
DEPS = SOURCES + ["planner.h", "kernels.cuh", "launch.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _source_hash(extra=()):
    """sha256 over every source the library is built from, the public header, this script and
    the nvcc flags: a prebuilt librexi.so is reused only if it was built from exactly these."""
    h = hashlib.sha256()
    files = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "rexi.h"),
                                                     os.path.abspath(__file__)]
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(FLAGS + list(extra)).encode())
    return h.hexdigest()


def _stale(lib, digest):
    stamp = lib + ".stamp"
    if not os.path.exists(lib) or not os.path.exists(stamp):
        return True
    with open(stamp) as f:
        return f.read().strip() != digest


def _build(lib, extra, force, verbose, log_name):
    digest = _source_hash(extra)
    if not force and not _stale(lib, digest):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *extra, "-shared", "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = r.stdout + r.stderr
    with open(os.path.join(HERE, log_name), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + log[-6000:])
    if verbose:
        print(log)
    os.replace(tmp, lib)
    with open(lib + ".stamp", "w") as f:
        f.write(digest + "\n")
    return lib


def build(force=False, verbose=False):
    return _build(LIB, [], force, verbose, "build.log")


def build_checked(force=False, verbose=False):
    """librexi_checked.so: the same sources with -DREXI_CHECKED."""
    return _build(LIB_CHECKED, ["-DREXI_CHECKED"], force, verbose, "build_checked.log")


if __name__ == "__main__":
    if "--checked" in sys.argv:
        build_checked(force="--force" in sys.argv, verbose=True)
    else:
        build(force="--force" in sys.argv, verbose=True)
