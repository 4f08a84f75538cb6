import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built librexi.so")
    config.addinivalue_line("markers", "slow: long-running oracle check")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import lrsw
    lrsw.build()
    return lrsw.lib()


def read_appendix_a():
    mu = None
    rows = []
    with open(os.path.join(GOLDEN, "appendix_a.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if parts[0] == "mu":
                mu = parts[1]
            else:
                rows.append((int(parts[0]), parts[1], parts[2]))
    return mu, rows


def read_paper_tables():
    rows = []
    with open(os.path.join(GOLDEN, "paper_tables.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            p = line.split()
            rows.append(dict(method=p[0], scenario=p[1], tau=float(p[2]), h=float(p[3]),
                             M=int(p[4]), paper=float(p[5]), cite=" ".join(p[6:])))
    return rows
