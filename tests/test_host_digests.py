"""CPU: the host-side digests of the product library (no device involved):
the SHA-NI SHA-256 used for load_group's model-file check (src/engine.cpp:79)
and hash_ops (src/messages.cpp:197-202) over request op lists, against
hashlib, the oracle restatement and the compiled reference."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden, split_reqs


def test_host_sha256_matches_hashlib():
    from paper_2205_15757_b200 import host_sha256
    rng = np.random.default_rng(1)
    for n in (0, 1, 55, 56, 63, 64, 65, 119, 120, 127, 128, 1000, 65537, 3_000_001):
        m = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert host_sha256(m) == hashlib.sha256(m).digest(), n


def test_host_sha256_scalar_path_matches():
    """CREDO_HOST_SHA_SCALAR=1 forces the portable round function (hosts
    without SHA-NI): same digests."""
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r);"
            "from paper_2205_15757_b200 import host_sha256, lib;"
            "assert lib().cg_host_sha_accelerated() == 0;"
            "rng = np.random.default_rng(2);"
            "ms = [rng.integers(0, 256, n, dtype=np.uint8).tobytes() for n in (0, 3, 64, 100, 9999)];"
            "assert all(host_sha256(m) == hashlib.sha256(m).digest() for m in ms)" % ROOT)
    env = dict(os.environ, CREDO_HOST_SHA_SCALAR="1")
    subprocess.run([sys.executable, "-c", code], check=True, env=env)


def _ops_case():
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_full.npz")
    reqs = split_reqs(g)
    rng = np.random.default_rng(3)
    cases = []
    for B in (1, 7, 64):
        idx = rng.choice(len(reqs), B, replace=False)
        encs = [reqs[i] for i in idx]
        versions = rng.integers(1, 2**40, B)
        statuses = (rng.random(B) < 0.2).astype(np.uint8)
        reasons = ["quorum unsatisfied" if s else "" for s in statuses]
        cases.append((encs, RequestBatch.from_encoded(encs), versions, statuses, reasons))
    return cases, g["gid"].tobytes()


def test_hash_ops_vs_oracle_and_reference(oracle):
    from oracle.oracle import Reference
    from paper_2205_15757_b200 import hash_ops_batches
    cases, gid = _ops_case()
    got = hash_ops_batches([c[1] for c in cases], gid, [c[2] for c in cases],
                           [c[3] for c in cases], [c[4] for c in cases], threads=3)
    for (encs, _, ver, st, rs), h in zip(cases, got):
        assert h == oracle.hash_ops(encs, ver, st, rs)
        if Reference.available():
            assert h == Reference().hash_ops(encs, ver, st, rs)
    # one version for every op, all ok
    encs, b = cases[1][0], cases[1][1]
    (h,) = hash_ops_batches([b], gid, [5])
    assert h == oracle.hash_ops(encs, [5] * len(encs), [0] * len(encs))


def test_hash_ops_threads_equal_serial():
    from paper_2205_15757_b200 import hash_ops_batches
    cases, gid = _ops_case()
    bs = [c[1] for c in cases] * 3
    vs = [1] * len(bs)
    assert hash_ops_batches(bs, gid, vs, threads=1) == hash_ops_batches(bs, gid, vs, threads=8)
