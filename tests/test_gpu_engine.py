"""GPU: the batch former in front of the device groups (cg_engine_*), against
the reference's own engine tests (proj/tests/test_engine.cpp:200-300) and
semantics (proj/src/engine.cpp:166-267): batches of exec_batch_max, the
flush deadline, one batch per live version, duplicate absorption, structural
request checks, unknown / retired groups, misfit requests -- and the batches
it forms certify to the reference's golden certificate."""
import numpy as np
import pytest

from conftest import golden, split_reqs

pytestmark = pytest.mark.gpu


def _models(ctx, g):
    from paper_2205_15757_b200 import Model
    return [Model.load_linear(ctx, g["files"][p].tobytes(), g["digests"][p].tobytes())
            for p in range(int(g["N"]))]


def _group(ctx, g, models, version=1, max_batch=16):
    from paper_2205_15757_b200 import EUCLIDEAN, ModelGroup
    return ModelGroup(ctx, models, 1, EUCLIDEAN, float(g["eps"]), g["gid"].tobytes(), version,
                      max_batch=max_batch, topk=3)


@pytest.fixture(scope="module")
def c1(ctx):
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_batch.npz")
    ms = _models(ctx, g)
    reqs = split_reqs(g)
    yield dict(g=g, models=ms, reqs=reqs, batch=RequestBatch.from_encoded(reqs))
    for m in ms:
        m.free()


def _sub(batch, idx):
    from paper_2205_15757_b200 import RequestBatch
    return RequestBatch(batch.request_ids[idx], batch.inputs[idx], batch.client_pubs[idx],
                        [batch.nonces[i] for i in idx], batch.client_sigs[idx],
                        None if batch.eps is None else [batch.eps[i] for i in idx])


def test_eight_requests_batch_max_four_form_two_batches(ctx, c1):
    """test_engine.cpp:220-243."""
    from paper_2205_15757_b200 import InferenceEngine
    grp = _group(ctx, c1["g"], c1["models"])
    eng = InferenceEngine(ctx, 4, 2000)
    eng.load_group(grp)
    for i in range(8):
        assert eng.submit(_sub(c1["batch"], [i]), 100 * i) == [0]
    ready = eng.ready()
    assert [r[3] for r in ready] == [4, 4]
    assert eng.next_flush_deadline() is None  # queues drained
    for grp_, ver, t, B in ready:
        r = grp_.certify_ticket(t, B=B)
        assert r["satisfied"].all()
    eng.free()
    grp.free()


def test_partial_batch_flushes_after_interval(ctx, c1):
    """test_engine.cpp:245-263."""
    from paper_2205_15757_b200 import InferenceEngine
    grp = _group(ctx, c1["g"], c1["models"])
    eng = InferenceEngine(ctx, 4, 5000)
    eng.load_group(grp)
    assert eng.submit(_sub(c1["batch"], [0]), 1000) == [0]
    assert eng.ready() == []
    assert eng.next_flush_deadline() == 6000
    eng.flush_due(5999)
    assert eng.ready() == []
    eng.flush_due(6000)
    ready = eng.ready()
    assert len(ready) == 1 and ready[0][3] == 1
    grp.certify_ticket(ready[0][2], B=1)
    eng.free()
    grp.free()


def test_multi_version_one_batch_per_live_version(ctx, c1):
    """test_engine.cpp:265-294: with v1 and v2 live (v2 defined), a
    submission forms one batch per version; each certifies under its own
    version; retiring v1 leaves v2 only; retiring both -> 'group retired'."""
    from paper_2205_15757_b200 import (GROUP_DEFINED, GROUP_RETIRED, SUBMIT_RETIRED,
                                       InferenceEngine)
    g1 = _group(ctx, c1["g"], c1["models"], version=1)
    g2 = _group(ctx, c1["g"], c1["models"], version=2)
    eng = InferenceEngine(ctx, 1, 2000)  # instant batches
    eng.load_group(g1)
    eng.load_group(g2, GROUP_DEFINED)
    assert eng.submit(_sub(c1["batch"], [3]), 0) == [0]
    ready = eng.ready()
    assert sorted(r[1] for r in ready) == [1, 2]
    roots = {}
    for grp_, ver, t, B in ready:
        r = grp_.certify_ticket(t, B=B, want_outputs=True)
        assert grp_.version == ver and r["satisfied"].all()
        roots[ver] = r["a_root"].tobytes()
    assert roots[1] != roots[2]  # the version is inside every leaf
    gid = c1["g"]["gid"].tobytes()
    eng.set_status(gid, 1, GROUP_RETIRED)
    assert eng.submit(_sub(c1["batch"], [4]), 0) == [0]
    assert [r[1] for r in eng.ready()] == [2]
    eng.set_status(gid, 2, GROUP_RETIRED)
    assert eng.submit(_sub(c1["batch"], [5]), 0) == [SUBMIT_RETIRED]
    eng.free()
    g1.free()
    g2.free()


def test_duplicates_absorbed_and_errors(ctx, c1):
    """Duplicate submissions are absorbed (test_engine.cpp:296-...);
    verify_request's structural checks and unknown groups are errors
    (test_engine.cpp:200-218)."""
    from paper_2205_15757_b200 import (SUBMIT_INVALID, SUBMIT_OK, SUBMIT_UNKNOWN_GROUP,
                                       InferenceEngine)
    grp = _group(ctx, c1["g"], c1["models"])
    eng = InferenceEngine(ctx, 4, 2000)
    eng.load_group(grp)
    b = c1["batch"]
    assert eng.submit(_sub(b, [0, 0, 1, 1, 0]), 0) == [SUBMIT_OK] * 5
    assert eng.pending() == (2, 0)
    assert eng.submit(_sub(b, [2]), 0, group_id=b"nope") == [SUBMIT_UNKNOWN_GROUP]
    forged = _sub(b, [6])
    forged.nonces = [forged.nonces[0] + b"x"]  # request id != canonical id
    assert eng.submit(forged, 0) == [SUBMIT_INVALID]
    empty = _sub(b, [7])
    empty.nonces = [b""]
    assert eng.submit(empty, 0) == [SUBMIT_INVALID]
    eng.flush_all()
    ((_, _, t, B),) = eng.ready()
    assert B == 2
    grp.certify_ticket(t, B=B)
    eng.free()
    grp.free()


def test_engine_batches_certify_to_the_golden(ctx, c1):
    """The whole 12-request golden batch through the batch former (batch max
    12, pack threads) certifies to the reference's certificate."""
    from paper_2205_15757_b200 import InferenceEngine
    g = c1["g"]
    grp = _group(ctx, g, c1["models"])
    eng = InferenceEngine(ctx, int(g["B"]), 2000, pack_threads=4)
    eng.load_group(grp)
    assert eng.submit(c1["batch"], 0) == [0] * int(g["B"])
    ((_, _, t, B),) = eng.ready()
    r = grp.certify_ticket(t, B=B, want_leaves=True)
    assert np.array_equal(r["leaf_hashes"], g["leaf_hashes"])
    assert np.array_equal(r["r_roots"], g["honest_r_roots"])
    assert np.array_equal(r["a_root"], g["honest_a_root"])
    eng.free()
    grp.free()


def test_engine_misfit_requests(ctx):
    """Wrong-dimension requests are queued like any other (submit does not
    check dims) and certified as misfits (c1_misfit.npz, from the reference)."""
    from paper_2205_15757_b200 import InferenceEngine, RequestBatch
    g = golden("c1_misfit.npz")
    ms = _models(ctx, g)
    grp = _group(ctx, g, ms)
    eng = InferenceEngine(ctx, int(g["B"]), 2000)
    eng.load_group(grp)
    batch = RequestBatch.from_encoded(split_reqs(g))
    assert eng.submit(batch, 0) == [0] * int(g["B"])
    ((_, _, t, B),) = eng.ready()
    r = grp.certify_ticket(t, B=B)
    assert np.array_equal(r["r_roots"], g["r_roots"])
    assert np.array_equal(r["a_root"], g["a_root"])
    eng.free()
    grp.free()
    for m in ms:
        m.free()
