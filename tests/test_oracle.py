"""CPU: the plain-C oracle restatement pinned against the reference's own
answers (golden fixtures generated from the compiled reference) and, where
oracle/_ref was built, against the live reference."""
import hashlib

import numpy as np
import pytest

from conftest import golden, split_reqs


def _msgs(g):
    data, lens = g["data"].tobytes(), g["lens"]
    out, off = [], 0
    for n in lens:
        out.append(data[off:off + int(n)])
        off += int(n)
    return out


def test_sha256_kats(oracle):
    # tests/test_codec.cpp:123-130 of the reference
    assert oracle.sha256(b"").hex() == (
        "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855")
    assert oracle.sha256(b"abc").hex() == (
        "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad")


def test_sha256_golden(oracle):
    g = golden("sha256.npz")
    for m, d in zip(_msgs(g), g["digests"]):
        assert oracle.sha256(m) == d.tobytes()
        assert hashlib.sha256(m).digest() == d.tobytes()
    assert oracle.sha256(b"a" * 1000000) == g["million_a"].tobytes()


def test_midstate_matches_streaming(oracle):
    msg = bytes(range(256)) * 3
    st = oracle.midstate(msg, 5)
    assert st.shape == (8,)
    # SHA of the message == compress(rest) from midstate: cross-check through
    # oracle.sha256 of the whole message vs hashlib
    assert oracle.sha256(msg) == hashlib.sha256(msg).digest()


def test_merkle_golden(oracle):
    g = golden("merkle.npz")
    lh = g["leaf_hashes"]
    data, lens = g["leaf_data"].tobytes(), g["leaf_lens"]
    off = i = 0
    for t, n in enumerate(g["counts"]):
        leaves = []
        for _ in range(int(n)):
            leaf = data[off:off + int(lens[i])]
            assert oracle.leaf_hash(leaf) == lh[i].tobytes()
            leaves.append(lh[i].tobytes())
            off += int(lens[i])
            i += 1
        assert oracle.merkle_root(leaves) == g["roots"][t].tobytes()
    with pytest.raises(ValueError):
        oracle.merkle_root([])


def test_merkle_formulas(oracle):
    # tests/test_merkle.cpp:51-69: 1-leaf root is the leaf hash; 2-leaf root
    # is H(0x01 || L || R); promotion is not duplication (:147-152)
    a, b, c = (oracle.leaf_hash(x) for x in (b"a", b"b", b"c"))
    assert oracle.merkle_root([a]) == a
    assert oracle.merkle_root([a, b]) == hashlib.sha256(b"\x01" + a + b).digest()
    ab = hashlib.sha256(b"\x01" + a + b).digest()
    assert oracle.merkle_root([a, b, c]) == hashlib.sha256(b"\x01" + ab + c).digest()
    assert oracle.merkle_root([a, b, c]) != oracle.merkle_root([a, b, c, c])


def test_select_quorum_golden(oracle):
    g = golden("quorum.npz")
    for t in range(len(g["n"])):
        n, f, dim, metric = (int(g[k][t]) for k in ("n", "f", "dim", "metric"))
        pres = int(g["present"][t])
        idx = [i for i in range(n) if pres >> i & 1]
        outs = g["outs"][t][idx][:, :dim]
        mask, diam, sat = oracle.select_quorum(outs, idx, n, f, metric, float(g["eps"][t]))
        assert mask == int(g["selected"][t]), t
        assert sat == bool(g["satisfied"][t]), t
        assert diam == float(g["diameter"][t]), t  # bit-exact
        if sat:
            lab = oracle.ensemble_label(g["outs"][t][:n, :dim], mask, f)
            assert lab == int(g["label"][t]), t


def test_select_quorum_errors(oracle):
    # distance.cpp:141-165: fewer than N-f present, f >= n -> invalid_argument
    with pytest.raises(ValueError):
        oracle.select_quorum(np.ones((2, 1)), [0, 1], 4, 1, 0, 1.0)
    with pytest.raises(ValueError):
        oracle.select_quorum(np.ones((3, 1)), [0, 1, 2], 3, 3, 0, 1.0)


@pytest.mark.parametrize("fixture", ["c1_batch.npz", "c1_full.npz"])
def test_c1_golden_linear_and_leaves(oracle, fixture):
    """c1_full.npz is C1 at SURVEY §8(d)'s shape (3072 -> 10 softmax, batch
    64, seed 7); c1_batch.npz the small variant (512 -> 10, batch 12)."""
    from oracle.oracle import parse_linear_model_file, parse_request
    g = golden(fixture)
    N, B, v = int(g["N"]), int(g["B"]), int(g["v"])
    reqs = split_reqs(g)
    gid = g["gid"].tobytes()
    inputs = [parse_request(r)["input"] for r in reqs]
    for p in range(N):
        u, v_, sm, W, b = parse_linear_model_file(g["files"][p].tobytes())
        assert sm == (fixture == "c1_full.npz") and v_ == v and u == int(g["u"])
        assert hashlib.sha256(g["files"][p].tobytes()).digest() == g["digests"][p].tobytes()
        for k in range(B):
            y = oracle.linear_run(W, b, inputs[k], sm)
            if sm:  # exp: the restatement uses the same libm as the reference build
                assert np.array_equal(y, g["outputs"][p, k]), (p, k)
            else:
                assert np.array_equal(y, g["outputs"][p, k])  # bit-exact fp64
    for k in range(B):
        f = parse_request(reqs[k])
        enc = oracle.request_encode(f["request_id"], f["group_id"], f["input"],
                                    f["eps"], f["pub"], f["nonce"], f["sig"])
        assert enc == reqs[k]
        for p in range(N):
            res = oracle.result_encode(f["request_id"], p, gid, 1,
                                       g["outputs"][p, k], g["digests"][p].tobytes())
            assert oracle.tagged_leaf_hash(0x52, enc, res) == g["leaf_hashes"][p, k].tobytes()


@pytest.mark.parametrize("variant", ["honest", "partial_fault", "failure"])
@pytest.mark.parametrize("fixture", ["c1_batch.npz", "c1_full.npz"])
def test_c1_golden_certify(oracle, variant, fixture):
    """Oracle restatement of the whole batch certification == reference."""
    from oracle.oracle import parse_request
    g = golden(fixture)
    N, B, eps = int(g["N"]), int(g["B"]), float(g["eps"])
    gid = g["gid"].tobytes()
    reqs = split_reqs(g)
    outs = g[f"{variant}_outputs"]
    sels, sats = [], []
    for k in range(B):
        f = parse_request(reqs[k])
        e = f["eps"] if f["eps"] is not None else eps
        mask, diam, sat = oracle.select_quorum(outs[:, k], list(range(N)), N, 1, 0, e)
        assert mask == int(g[f"{variant}_sel"][k])
        assert diam == float(g[f"{variant}_diam"][k])
        assert sat == bool(g[f"{variant}_sat"][k])
        lab = oracle.ensemble_label(outs[:, k], mask, 1) if sat else -1
        assert lab == int(g[f"{variant}_label"][k])
        sels.append(mask)
        sats.append(sat)
    # R roots from leaf hashes over this variant's outputs
    leaves = {}
    for p in range(N):
        hs = []
        for k in range(B):
            f = parse_request(reqs[k])
            res = oracle.result_encode(f["request_id"], p, gid, 1, outs[p, k],
                                       g["digests"][p].tobytes())
            hs.append(oracle.tagged_leaf_hash(0x52, reqs[k], res))
            leaves[(k, p)] = res
        assert oracle.merkle_root(hs) == g[f"{variant}_r_roots"][p].tobytes()
    man = oracle.attest_manifest(sels, sats, N)
    assert len(man) == int(g[f"{variant}_mlen"])
    a_leaves = []
    for kind, node, op in man:
        if kind == 0:
            a_leaves.append(oracle.leaf_hash(b"\x57" + g[f"{variant}_r_roots"][node].tobytes()))
        elif kind == 1:
            a_leaves.append(oracle.tagged_leaf_hash(0x53, reqs[op], leaves[(op, node)]))
        else:
            f = parse_request(reqs[op])
            a_leaves.append(oracle.leaf_hash(oracle.failure_leaf(f["request_id"], gid, 1)))
    assert oracle.merkle_root(a_leaves) == g[f"{variant}_a_root"].tobytes()


def test_live_reference_cross_check(oracle):
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built here")
    R = Reference()
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(3, 9))
        f = max(1, (n - 1) // 3)
        outs = rng.uniform(0, 1, (1, 7)) + rng.uniform(-0.05, 0.05, (n, 7)) * rng.choice([1, 40], (n, 1))
        e = float(rng.uniform(0, 0.3))
        assert oracle.select_quorum(outs, list(range(n)), n, f, 0, e) == \
            R.select_quorum(outs, list(range(n)), n, f, 0, e)
    for n in (0, 1, 63, 64, 65, 1000):
        m = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert oracle.sha256(m) == R.sha256(m)


@pytest.mark.parametrize("n,f,v,metric", [(4, 1, 6, 0), (8, 2, 6, 0), (5, 1, 4, 2),
                                          (8, 3, 3, 2), (3, 1, 1, 1), (3, 1, 4, 1),
                                          (2, 1, 4, 1)])
def test_adversarial_oracle_vs_reference(oracle, n, f, v, metric):
    """The C restatement against the compiled reference (select_quorum +
    ensemble_label) on the NaN/Inf/tie generator the GPU sweeps use, so the
    GPU-vs-oracle adversarial sweep is pinned to the reference itself;
    includes max_minus_min on vectors (throws only when delta runs, m >= 2,
    distance.cpp:87-91) and on single present results."""
    from adversarial import adversarial
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built here")
    R = Reference()
    rng = np.random.default_rng(n * 1000 + v * 10 + metric)
    outs = adversarial(rng, 400, n, v)
    eps = rng.choice([0.0, 0.1, 0.25, 1.0], 400)
    for k in range(400):
        for idx in (list(range(n)), [0], list(range(1, n))):
            want = got = None
            try:
                want = R.select_quorum(outs[k][idx], idx, n, f, metric, eps[k])
            except ValueError:
                want = "throws"
            try:
                got = oracle.select_quorum(outs[k][idx], idx, n, f, metric, eps[k])
            except ValueError:
                got = "throws"
            assert got == want or (isinstance(got, tuple) and got[:1] + got[2:] == want[:1] + want[2:]
                                   and np.array_equal(np.float64(got[1]).view(np.uint64),
                                                      np.float64(want[1]).view(np.uint64))), (k, idx)
            if isinstance(want, tuple) and want[2]:
                assert oracle.ensemble_label(outs[k][idx], want[0], f) == \
                    R.ensemble_label(outs[k][idx], want[0], f)


def test_c1_misfit_golden(oracle):
    """Misfit requests (wrong input dimension): missing_result_leaf in every
    R tree, unsatisfied, a failure leaf -- the oracle restatement against the
    reference's answers (c1_misfit.npz)."""
    from oracle.oracle import parse_request
    g = golden("c1_misfit.npz")
    N, B, eps = int(g["N"]), int(g["B"]), float(g["eps"])
    gid = g["gid"].tobytes()
    reqs = split_reqs(g)
    miss = g["missing"].astype(bool)
    sels, sats, leaves = [], [], {}
    for k in range(B):
        if miss[k]:
            m, d, sat = 0, 0.0, False
        else:
            m, d, sat = oracle.select_quorum(g["outputs"][:, k], list(range(N)), N, 1, 0, eps)
        assert (m, sat) == (int(g["sel"][k]), bool(g["sat"][k]))
        sels.append(m)
        sats.append(sat)
    for p in range(N):
        hs = []
        for k in range(B):
            f = parse_request(reqs[k])
            assert len(f["input"]) == int(g["dims"][k])
            if miss[k]:
                hs.append(oracle.tagged_leaf_hash(0x4D, reqs[k], b""))
            else:
                res = oracle.result_encode(f["request_id"], p, gid, 1, g["outputs"][p, k],
                                           g["digests"][p].tobytes())
                leaves[(k, p)] = res
                hs.append(oracle.tagged_leaf_hash(0x52, reqs[k], res))
        assert oracle.merkle_root(hs) == g["r_roots"][p].tobytes()
    man = oracle.attest_manifest(sels, sats, N)
    assert len(man) == int(g["mlen"])
    a = []
    for kind, node, op in man:
        if kind == 1:
            a.append(oracle.tagged_leaf_hash(0x53, reqs[op], leaves[(op, node)]))
        else:
            assert kind == 2
            rid = parse_request(reqs[op])["request_id"]
            a.append(oracle.leaf_hash(oracle.failure_leaf(rid, gid, 1)))
    assert oracle.merkle_root(a) == g["a_root"].tobytes()


def test_c1_slot_golden(oracle):
    """The mixed op list (c1_slot.npz): the oracle's leaf constructions and
    fold reproduce the reference's R roots, manifest and A root --
    0x52 / 0x4D / 0x47 R leaves, outcomes only for ok request ops, failure
    leaves from the ops' own FailureRecord bytes."""
    from oracle.oracle import parse_request
    g = golden("c1_slot.npz")
    N, B, eps = int(g["N"]), int(g["B"]), float(g["eps"])
    gid = g["gid"].tobytes()
    kinds = g["kinds"]
    lens, buf = g["req_lens"], g["reqs"].tobytes()
    reqs, off = [], 0
    for n in lens:
        reqs.append(buf[off:off + int(n)])
        off += int(n)
    ents, recs, o1, o2 = [], [], 0, 0
    for a, b in zip(g["entry_lens"], g["rec_lens"]):
        ents.append(g["entries"].tobytes()[o1:o1 + int(a)])
        recs.append(g["recs"].tobytes()[o2:o2 + int(b)])
        o1 += int(a)
        o2 += int(b)
    sels, sats, res = {}, {}, {}
    for k in range(B):
        if kinds[k] == 0:
            m, d, s_ = oracle.select_quorum(g["outputs"][:, k], list(range(N)), N, 1, 0, eps)
            sels[k], sats[k] = m, s_
    for p in range(N):
        hs = []
        for k in range(B):
            if kinds[k] == 0:
                f = parse_request(reqs[k])
                res[(k, p)] = oracle.result_encode(f["request_id"], p, gid, 1,
                                                   g["outputs"][p, k], g["digests"][p].tobytes())
                hs.append(oracle.tagged_leaf_hash(0x52, reqs[k], res[(k, p)]))
            elif kinds[k] == 1:
                hs.append(oracle.tagged_leaf_hash(0x4D, reqs[k], b""))
            else:
                hs.append(oracle.leaf_hash(b"\x47" + ents[k]))
        assert oracle.merkle_root(hs) == g["r_roots"][p].tobytes(), p
    whole = [p for p in range(N) if all(sats[k] and sels[k] >> p & 1 for k in sats)]
    a = [oracle.leaf_hash(b"\x57" + g["r_roots"][p].tobytes()) for p in whole]
    for k in sorted(sats):
        if sats[k]:
            for p in range(N):
                if sels[k] >> p & 1 and p not in whole:
                    a.append(oracle.tagged_leaf_hash(0x53, reqs[k], res[(k, p)]))
    for k in range(B):
        if kinds[k] == 0 and not sats[k]:
            rid = parse_request(reqs[k])["request_id"]
            a.append(oracle.leaf_hash(oracle.failure_leaf(rid, gid, 1)))
        elif recs[k]:
            a.append(oracle.leaf_hash(b"\x46" + recs[k]))
    assert len(a) == int(g["mlen"])
    assert oracle.merkle_root(a) == g["a_root"].tobytes()


def test_label_digest_layout(oracle):
    """The compact agreed-label digest (new, C5 'D2') is plain SHA-256 over
    0x4C || id || u64be version || u64be label; pinned by the SHA KATs."""
    import hashlib
    rng = np.random.default_rng(9)
    for label in (-1, 0, 7, 999, 2**40):
        rid = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
        want = hashlib.sha256(b"\x4c" + rid + (3).to_bytes(8, "big")
                              + label.to_bytes(8, "big", signed=True)).digest()
        assert oracle.label_digest(rid, 3, label) == want


def test_agree_batch_matches_per_request(oracle):
    rng = np.random.default_rng(10)
    n, R, v = 5, 40, 7
    outs = rng.random((n, R, v))
    outs[rng.random((n, R)) < 0.2] += 0.5
    eps = rng.choice([0.2, 0.6, 1.0], R)
    ids = rng.integers(0, 256, (R, 32), dtype=np.uint8)
    r = oracle.agree_batch(outs, 1, 0, eps, ids, version=2)
    for k in range(R):
        mask, diam, sat = oracle.select_quorum(outs[:, k], np.arange(n), n, 1, 0, eps[k])
        assert (mask, diam, sat) == (int(r["selected"][k]), r["diameter"][k], r["satisfied"][k])
        lab = oracle.ensemble_label(outs[:, k], mask, 1) if sat else -1
        assert lab == r["label"][k]
        assert r["digest"][k].tobytes() == oracle.label_digest(ids[k].tobytes(), 2, lab)


def test_perturb_golden(oracle):
    """oc_perturb == PerturbingExecutor::run (model.cpp:75-105) bit-exact on
    the compiled reference's outputs (tests/golden/perturb.npz)."""
    g = golden("perturb.npz")
    for c in range(int(g["ncases"])):
        u, v, sm, node = (int(t) for t in g[f"c{c}_case"])
        mag = float(g[f"c{c}_mag"])
        dig = g[f"c{c}_digest"].tobytes()
        for k, x in enumerate(g[f"c{c}_inputs"]):
            y = oracle.perturb(node, dig, x, g[f"c{c}_plain"][k], mag)
            assert np.array_equal(y, g[f"c{c}_outputs"][k]), (c, k)


def test_perturb_live_reference(oracle):
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built here")
    R = Reference()
    files, digs = R.generate_group(b"group-0", 17, 4, 1, 0, 0.05, 21)
    x = np.random.default_rng(3).uniform(-1, 1, (3, 17))
    with pytest.raises(ValueError):
        R.perturbing_run(files[0], x, 4, 0, -1.0)
    with pytest.raises(ValueError):
        R.perturbing_run(files[0], x, 4, 0, float("nan"))
    plain = R.linear_run(files[0], x, 4)
    for node in (0, 1, 2**63):
        want = R.perturbing_run(files[0], x, 4, node, 0.125)
        got = np.stack([oracle.perturb(node, digs[0], x[k], plain[k], 0.125) for k in range(3)])
        assert np.array_equal(got, want)
