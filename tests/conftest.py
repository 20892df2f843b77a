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


def check_certificate(r, batch, digests, f, default_eps, gid, oracle, version=1, topk=5):
    """Every decision and digest of a certify() result recomputed by the
    oracle from the GPU's own per-replica outputs."""
    from paper_2205_15757_b200 import EUCLIDEAN
    from paper_2205_15757_b200.workload import encode_request
    outs = r["outputs"]
    N, B = outs.shape[0], outs.shape[1]
    sels, sats = [], []
    for k in range(B):
        e = default_eps if batch.eps is None or batch.eps[k] is None else batch.eps[k]
        m, d, s = oracle.select_quorum(outs[:, k], list(range(N)), N, f, EUCLIDEAN, e)
        assert (int(r["selected"][k]), float(r["diameter"][k]), bool(r["satisfied"][k])) == (m, d, s)
        lab = oracle.ensemble_label(outs[:, k], m, f) if s else -1
        assert int(r["label"][k]) == lab
        sels.append(m)
        sats.append(s)
        for p in range(N):
            idx, val = oracle.topk(outs[p, k], topk)
            assert np.array_equal(r["topk_idx"][p, k], idx)
    leaves = {}
    for p in range(N):
        hs = []
        for k in range(B):
            req = encode_request(batch, k, gid)
            res = oracle.result_encode(batch.request_ids[k].tobytes(), p, gid, version,
                                       outs[p, k], digests[p])
            h = oracle.tagged_leaf_hash(0x52, req, res)
            assert r["leaf_hashes"][p, k].tobytes() == h, (p, k)
            hs.append(h)
            leaves[(k, p)] = (req, res)
        assert r["r_roots"][p].tobytes() == oracle.merkle_root(hs)
    man = oracle.attest_manifest(sels, sats, N)
    assert int(r["manifest_len"][0]) == len(man)
    a = []
    for kind, node, op in man:
        if kind == 0:
            a.append(oracle.leaf_hash(b"\x57" + r["r_roots"][node].tobytes()))
        elif kind == 1:
            req, res = leaves[(op, node)]
            a.append(oracle.tagged_leaf_hash(0x53, req, res))
        else:
            a.append(oracle.leaf_hash(oracle.failure_leaf(batch.request_ids[op].tobytes(), gid,
                                                          version)))
    assert r["a_root"].tobytes() == oracle.merkle_root(a)
    return sels, sats
