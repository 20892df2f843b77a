"""GPU: cg_cert_leaf_hashes -- the leaves a verifier (verify_cert,
certificate.cpp:215-288) or a proxy (assemble_response, proxy.cpp:80-186)
re-hashes: leaf_hash(result_leaf) 0x52, leaf_hash(single_attest_leaf) 0x53
and leaf_hash(missing_result_leaf) 0x4D (messages.cpp:204-218, :283-290),
each request's prefix hashed once as a midstate. Checked bit-exact against
hashlib over the canonical request bytes (workload.encode_request, pinned to
the reference by the golden request leaves) and arbitrary result bytes,
including results shorter and longer than a block and the C2 input size."""
import hashlib

import numpy as np
import pytest

from paper_2205_15757_b200 import Context
from paper_2205_15757_b200.workload import encode_request, signed_requests

pytestmark = pytest.mark.gpu
TAG = {1: b"\x52", 2: b"\x53", 4: b"\x4d"}


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def expected(batch, gid, k, want, res):
    body = encode_request(batch, k, gid)
    if want == 4:
        return hashlib.sha256(b"\x00" + TAG[4] + body).digest()
    return hashlib.sha256(b"\x00" + TAG[want] + body + res).digest()


@pytest.mark.parametrize("B,u", [(5, 37), (3, 3 * 224 * 224)])
def test_cert_leaf_hashes(ctx, B, u):
    rng = np.random.default_rng(B * 7 + u)
    batch = signed_requests(B, u, seed=B)
    gid = b"group-0"
    ridx, want, res = [], [], []
    for m in range(4 * B):
        k = int(rng.integers(0, B))
        w = int(rng.choice([1, 2, 4]))
        n = int(rng.choice([0, 1, 55, 64, 175, 8095]))
        r = b"" if w == 4 else rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        ridx.append(k)
        want.append(w)
        res.append(r)
    h52, h53, h4d = ctx.cert_leaf_hashes(batch, gid, ridx, want, res)
    for m, (k, w, r) in enumerate(zip(ridx, want, res)):
        got = {1: h52, 2: h53, 4: h4d}[w][m].tobytes()
        assert got == expected(batch, gid, k, w, r), (m, k, w, len(r))


def test_cert_leaf_hashes_rejects_bad_input(ctx):
    batch = signed_requests(2, 8, seed=1)
    with pytest.raises(Exception):
        ctx.cert_leaf_hashes(batch, b"g", [2], [1], [b"x"])  # request index out of range
    with pytest.raises(Exception):
        ctx.cert_leaf_hashes(batch, b"g", [0], [8], [b"x"])  # want is a mask of 1 | 2 | 4
