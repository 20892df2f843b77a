import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libcredo_gpu.so")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ctx():
    from paper_2205_15757_b200 import Context
    c = Context(0)
    yield c
    c.close()


def split_reqs(g):
    lens = g["req_lens"]
    buf = g["reqs"].tobytes()
    out, off = [], 0
    for n in lens:
        out.append(buf[off:off + int(n)])
        off += int(n)
    return out
