"""GPU: verify_request's digests (domain.cpp:177-216) for a
batch -- signing digest SHA-256(0x01 || body), canonical request id, the
structural checks -- against the compiled reference (oracle/_ref) and an
independent hashlib restatement; the Ed25519 step (host) then accepts exactly
the requests the reference's verify_request accepts."""
import ctypes as C
import hashlib

import numpy as np
import pytest
from conftest import golden, split_reqs

pytestmark = pytest.mark.gpu


def test_signing_digests_c1_golden(ctx):
    from oracle.oracle import Reference
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_batch.npz")
    encs = split_reqs(g)
    b = RequestBatch.from_encoded(encs)
    sig, ids, st = ctx.request_digests(b, g["gid"].tobytes())
    R = Reference()
    for k, e in enumerate(encs):
        assert sig[k].tobytes() == R.signing_digest(e)
        assert sig[k].tobytes() == hashlib.sha256(b"\x01" + e[:-64]).digest()
        assert ids[k].tobytes() == b.request_ids[k].tobytes()
    assert not st.any()
    assert all(R.verify_request(e) == 1 for e in encs)


def test_signing_digests_imagenet_and_ed25519(ctx):
    from paper_2205_15757_b200.workload import _sodium, encode_request, signed_requests
    b = signed_requests(5, 3 * 224 * 224, seed=12, eps=[None, 0.3, None, None, 0.0])
    sig, ids, st = ctx.request_digests(b, b"group-0")
    L = _sodium()
    assert not st.any()
    for k in range(5):
        e = encode_request(b, k)
        assert sig[k].tobytes() == hashlib.sha256(b"\x01" + e[:-64]).digest()
        ok = L.crypto_sign_verify_detached(b.client_sigs[k].tobytes(), sig[k].tobytes(),
                                           C.c_ulonglong(32), b.client_pubs[k].tobytes())
        assert ok == 0  # libsodium: 0 = valid signature over the signing digest


def test_structural_checks(ctx):
    from copy import deepcopy

    from paper_2205_15757_b200.workload import signed_requests
    b = signed_requests(4, 12, seed=13, eps=[None, float("nan"), -1.0, None])
    b2 = deepcopy(b)
    b2.request_ids = np.array(b2.request_ids).copy()
    b2.request_ids[3, 0] ^= 1  # forged id
    _, _, st = ctx.request_digests(b2, b"group-0")
    assert list(st) == [0, 3, 3, 4]
