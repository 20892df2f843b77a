"""GPU parity: SHA-256 / leaf / Merkle kernels, select_quorum + label vote,
the fp64 LinearToyModel executor, and whole-batch certification — all through
the C-ABI, bit-exact against the oracle and the reference's golden vectors."""
import hashlib

import numpy as np
import pytest

from conftest import golden, split_reqs

pytestmark = pytest.mark.gpu


def _msgs(g):
    data, lens = g["data"].tobytes(), g["lens"]
    out, off = [], 0
    for n in lens:
        out.append(data[off:off + int(n)])
        off += int(n)
    return out


# ------------------------------------------------------------------ SHA-256
def test_sha256_golden(ctx):
    g = golden("sha256.npz")
    msgs = _msgs(g)
    got = ctx.hash_batch(msgs)
    for m, d, want in zip(msgs, got, g["digests"]):
        assert d == want.tobytes(), len(m)
    assert ctx.hash(b"a" * 1000000) == g["million_a"].tobytes()


def test_sha256_random_lengths(ctx, oracle):
    rng = np.random.default_rng(1)
    msgs = [rng.integers(0, 256, int(n), dtype=np.uint8).tobytes()
            for n in rng.integers(0, 3000, 500)]
    assert ctx.hash_batch(msgs) == [oracle.sha256(m) for m in msgs]


def test_leaf_hash_and_merkle_golden(ctx):
    g = golden("merkle.npz")
    data, lens = g["leaf_data"].tobytes(), g["leaf_lens"]
    leaves, off = [], 0
    for n in lens:
        leaves.append(data[off:off + int(n)])
        off += int(n)
    got = ctx.leaf_hash_batch(leaves)
    assert got == [h.tobytes() for h in g["leaf_hashes"]]
    trees, i = [], 0
    for n in g["counts"]:
        trees.append(got[i:i + int(n)])
        i += int(n)
    assert ctx.merkle_roots(trees) == [r.tobytes() for r in g["roots"]]


def test_merkle_large_tree(ctx, oracle):
    rng = np.random.default_rng(2)
    for n in (8191, 8192, 8193, 20001):
        leaves = [rng.integers(0, 256, 32, dtype=np.uint8).tobytes() for _ in range(n)]
        assert ctx.merkle_roots([leaves]) == [oracle.merkle_root(leaves)]


def test_merkle_empty_is_invalid(ctx):
    from paper_2205_15757_b200 import InvalidArgument
    with pytest.raises(InvalidArgument):
        ctx.merkle_roots([[]])


# --------------------------------------------------------------- agreement
def test_select_quorum_golden(ctx):
    g = golden("quorum.npz")
    T = len(g["n"])
    # group instances by (n, dim, metric, f) to batch them
    keys = {}
    for t in range(T):
        keys.setdefault((int(g["n"][t]), int(g["dim"][t]), int(g["metric"][t]),
                         int(g["f"][t])), []).append(t)
    for (n, dim, metric, f), ts in keys.items():
        outs = g["outs"][ts][:, :n, :dim]
        r = ctx.select_quorum_batch(outs, n, f, metric, g["eps"][ts],
                                    present=g["present"][ts])
        assert np.array_equal(r["selected"], g["selected"][ts].astype(np.uint32))
        assert np.array_equal(r["satisfied"], g["satisfied"][ts].astype(bool))
        assert np.array_equal(r["diameter"], g["diameter"][ts])  # bit-exact
        want_lab = np.where(g["satisfied"][ts] > 0, g["label"][ts], -1)
        assert np.array_equal(r["label"], want_lab)


def test_select_quorum_random_vs_oracle(ctx, oracle):
    rng = np.random.default_rng(7)
    for n, f, v in ((3, 1, 10), (4, 1, 1000), (8, 2, 1000), (7, 2, 3), (16, 5, 4)):
        R = 300 if v < 1000 else 60
        center = rng.uniform(0, 1, (R, 1, v))
        outs = center + rng.uniform(-0.01, 0.01, (R, n, v))
        shift = rng.random((R, n)) < 0.2
        outs = outs + shift[..., None] * 3 * 0.05 / np.sqrt(v)
        eps = np.full(R, 0.05 if v > 10 else 0.03)
        r = ctx.select_quorum_batch(outs, n, f, 0, eps)
        for k in range(R):
            m, d, s = oracle.select_quorum(outs[k], list(range(n)), n, f, 0, eps[k])
            assert (int(r["selected"][k]), float(r["diameter"][k]), bool(r["satisfied"][k])) == (m, d, s)
            lab = oracle.ensemble_label(outs[k], m, f) if s else -1
            assert int(r["label"][k]) == lab


def test_select_quorum_pinned_and_errors(ctx):
    from paper_2205_15757_b200 import EUCLIDEAN, InvalidArgument
    # tests/test_distance.cpp:138-160
    o = ctx.select_quorum({0: [1.00], 1: [1.01], 2: [1.02], 3: [5.0]}, 4, 1, EUCLIDEAN, 0.2)
    assert o.satisfied and o.selected == {0, 1, 2}
    o = ctx.select_quorum({i: [2.0] for i in range(4)}, 4, 1, EUCLIDEAN, 0.0)
    assert o.satisfied and o.selected == {0, 1, 2, 3} and o.diameter == 0.0
    o = ctx.select_quorum({0: [1.0], 1: [1.5], 2: [2.0], 3: [2.5]}, 4, 1, EUCLIDEAN, 0.2)
    assert not o.satisfied and o.selected == set()
    with pytest.raises(InvalidArgument):
        ctx.select_quorum({0: [1.0], 1: [1.0]}, 4, 1, EUCLIDEAN, 1.0)


# ---------------------------------------------------------- executor seam
def test_linear_executor_bit_exact(ctx):
    from oracle.oracle import parse_linear_model_file
    from paper_2205_15757_b200 import CudaExecutor, DigestMismatch, Model
    g = golden("c1_batch.npz")
    ex = CudaExecutor(ctx)
    for p in range(int(g["N"])):
        m = Model.load_linear(ctx, g["files"][p].tobytes(), g["digests"][p].tobytes())
        y = ex.run(m, g["inputs"])
        assert np.array_equal(y, g["outputs"][p])  # LinearToyModel::run, fp64
        m.free()
    bad = bytearray(g["digests"][0].tobytes())
    bad[0] ^= 1
    with pytest.raises(DigestMismatch):
        Model.load_linear(ctx, g["files"][0].tobytes(), bytes(bad))


def test_linear_softmax_within_ulp(ctx, oracle):
    from oracle.oracle import parse_linear_model_file
    from paper_2205_15757_b200 import CudaExecutor, Model
    g = golden("c1_batch.npz")
    f = bytearray(g["files"][0].tobytes())
    f[16] = 1  # softmax flag byte (model.cpp:38-46)
    f = bytes(f)
    m = Model.load_linear(ctx, f, hashlib.sha256(f).digest())
    u, v, sm, W, b = parse_linear_model_file(f)
    y = CudaExecutor(ctx).run(m, g["inputs"])
    want = np.stack([oracle.linear_run(W, b, x, True) for x in g["inputs"]])
    # exp() differs by <= 1 ulp between CUDA and glibc; stated tolerance 4 ulp
    assert np.all(np.abs(y - want) <= 4 * np.spacing(want))


# ------------------------------------------------------ whole-batch certify
def _group(ctx, g, B):
    from paper_2205_15757_b200 import EUCLIDEAN, Model, ModelGroup
    models = [Model.load_linear(ctx, g["files"][p].tobytes(), g["digests"][p].tobytes())
              for p in range(int(g["N"]))]
    return ModelGroup(ctx, models, 1, EUCLIDEAN, float(g["eps"]),
                      g["gid"].tobytes(), 1, max_batch=B, topk=3)


def test_certify_batch_c1_bit_exact(ctx):
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_batch.npz")
    B = int(g["B"])
    grp = _group(ctx, g, B)
    batch = RequestBatch.from_encoded(split_reqs(g))
    r = grp.certify(batch, want_outputs=True, want_leaves=True)
    assert np.array_equal(r["outputs"], g["outputs"])
    assert np.array_equal(r["leaf_hashes"], g["leaf_hashes"])
    assert np.array_equal(r["selected"], g["honest_sel"].astype(np.uint32))
    assert np.array_equal(r["diameter"], g["honest_diam"])
    assert np.array_equal(r["satisfied"], g["honest_sat"].astype(bool))
    assert np.array_equal(r["label"], g["honest_label"])
    assert np.array_equal(r["r_roots"], g["honest_r_roots"])
    assert np.array_equal(r["a_root"], g["honest_a_root"])
    assert int(r["manifest_len"][0]) == int(g["honest_mlen"])
    # top-1 of each replica output == argmax
    assert np.array_equal(r["topk_idx"][..., 0], np.argmax(g["outputs"], axis=-1))


def test_certify_c1_full_shape(ctx, oracle):
    """C1 at SURVEY §8(d)'s shape (c1_full.npz: generate_group 3072 -> 10
    with softmax, 3 replicas, f=1, batch 64, seed 7, from the compiled
    reference): the GPU's softmax outputs within the stated 4 ulp of the
    reference's (CUDA exp vs glibc exp), every digest and decision recomputed
    by the oracle from the GPU's own outputs, and the reference's own
    certificates (roots, manifests) reproduced bit-exact from its outputs for
    the honest / fault / failure variants."""
    from conftest import check_certificate
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_full.npz")
    B, N = int(g["B"]), int(g["N"])
    grp = _group(ctx, g, B)
    batch = RequestBatch.from_encoded(split_reqs(g))
    r = grp.certify(batch, want_outputs=True, want_leaves=True)
    want = g["outputs"]
    assert np.all(np.abs(r["outputs"] - want) <= 4 * np.spacing(want))
    digs = [g["digests"][p].tobytes() for p in range(N)]
    check_certificate(r, batch, digs, 1, float(g["eps"]), g["gid"].tobytes(), oracle, topk=3)
    for variant in ("honest", "partial_fault", "failure"):
        r = grp.certify_outputs(batch, g[f"{variant}_outputs"])
        assert np.array_equal(r["selected"], g[f"{variant}_sel"].astype(np.uint32))
        assert np.array_equal(r["diameter"].view(np.uint64), g[f"{variant}_diam"].view(np.uint64))
        assert np.array_equal(r["satisfied"], g[f"{variant}_sat"].astype(bool))
        assert np.array_equal(r["label"], g[f"{variant}_label"])
        assert np.array_equal(r["r_roots"], g[f"{variant}_r_roots"])
        assert int(r["manifest_len"][0]) == int(g[f"{variant}_mlen"])
        assert np.array_equal(r["a_root"], g[f"{variant}_a_root"]), variant
    grp.free()


def test_certify_misfit_requests(ctx):
    """Requests whose input dimension differs from the group's: skipped by
    execute_batch (engine.cpp:286-291), so missing_result_leaf (0x4D) in every
    R tree, unsatisfied, failure leaves -- bit-exact against the compiled
    reference (c1_misfit.npz), through the whole GPU certify path."""
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_misfit.npz")
    B = int(g["B"])
    grp = _group(ctx, g, B)
    batch = RequestBatch.from_encoded(split_reqs(g))
    assert isinstance(batch.inputs, list)
    r = grp.certify(batch, want_outputs=True)
    fit = ~g["missing"].astype(bool)
    assert np.array_equal(r["outputs"][:, fit], g["outputs"][:, fit])
    assert np.array_equal(r["selected"], g["sel"].astype(np.uint32))
    assert np.array_equal(r["satisfied"], g["sat"].astype(bool))
    assert np.array_equal(r["label"][~fit], [-1, -1])
    assert np.array_equal(r["r_roots"], g["r_roots"])
    assert int(r["manifest_len"][0]) == int(g["mlen"])
    assert np.array_equal(r["a_root"], g["a_root"])
    grp.free()


def _slot_batch(g):
    """c1_slot.npz as a RequestBatch with its op-list structure: request ops
    carry their request fields, group ops zeros (ignored)."""
    from oracle.oracle import parse_request
    from paper_2205_15757_b200 import RequestBatch
    B, u = int(g["B"]), int(g["u"])
    lens, buf = g["req_lens"], g["reqs"].tobytes()
    ids, ins, pubs, nonces, sigs, eps, off = [], [], [], [], [], [], 0
    for k in range(B):
        n = int(lens[k])
        if n:
            f = parse_request(buf[off:off + n])
            ids.append(np.frombuffer(f["request_id"], np.uint8))
            ins.append(f["input"])
            pubs.append(np.frombuffer(f["pub"], np.uint8))
            nonces.append(f["nonce"])
            sigs.append(np.frombuffer(f["sig"], np.uint8))
            eps.append(f["eps"])
        else:
            ids.append(np.zeros(32, np.uint8))
            ins.append(np.zeros(u))
            pubs.append(np.zeros(32, np.uint8))
            nonces.append(b"")
            sigs.append(np.zeros(64, np.uint8))
            eps.append(None)
        off += n
    def split(data, ls):
        out, o = [], 0
        for n in ls:
            out.append(data[o:o + int(n)])
            o += int(n)
        return out
    kinds = g["kinds"].tolist()
    entries = split(g["entries"].tobytes(), g["entry_lens"])
    return RequestBatch(np.stack(ids), np.stack(ins), np.stack(pubs), nonces, np.stack(sigs),
                        eps if any(e is not None for e in eps) else None,
                        op_kinds=kinds,
                        op_entries=[e if kd == 2 else b"" for e, kd in zip(entries, kinds)],
                        fail_records=split(g["recs"].tobytes(), g["rec_lens"]))


def test_certify_mixed_slot(ctx):
    """A PRE-PREPARE op list mixing ok requests, rejected requests and
    activate_group ops (c1_slot.npz, from the compiled reference's
    build_result_tree + try_attest manifest): R leaves 0x52 / 0x4D / 0x47,
    outcomes only for ok request ops, explicit failure leaves -- bit-exact."""
    g = golden("c1_slot.npz")
    B = int(g["B"])
    grp = _group(ctx, g, B)
    batch = _slot_batch(g)
    r = grp.certify_outputs(batch, g["outputs"])
    assert np.array_equal(r["r_roots"], g["r_roots"])
    assert int(r["manifest_len"][0]) == int(g["mlen"])
    assert np.array_equal(r["a_root"], g["a_root"])
    assert np.array_equal(r["satisfied"], g["sat"].astype(bool))
    # and with the replicas' own forwards (the ok rows equal the fixture's
    # honest outputs except the injected fault on provider 2, op 5)
    r2 = grp.certify(batch, want_outputs=True)
    ok = g["kinds"] == 0
    got, want = r2["outputs"].copy(), g["outputs"].copy()
    got[2, 5] = want[2, 5] = 0.0  # the fixture's injected fault
    assert np.array_equal(got[:, ok], want[:, ok])
    grp.free()


def test_certify_empty_slot(ctx, oracle):
    """An empty filler slot (messages.cpp:240-243): noop R leaves, N
    whole-batch A leaves."""
    import struct
    g = golden("c1_slot.npz")
    grp = _group(ctx, g, 4)
    r = grp.certify_empty_slot(7, 42)
    leaf = oracle.leaf_hash(b"\x4e" + struct.pack(">QQ", 7, 42))
    assert all(x.tobytes() == leaf for x in r["r_roots"])
    a = oracle.leaf_hash(b"\x57" + leaf)
    assert r["a_root"].tobytes() == oracle.merkle_root([a] * int(g["N"]))
    assert int(r["manifest_len"][0]) == int(g["N"])
    grp.free()


@pytest.mark.parametrize("variant", ["honest", "partial_fault", "failure"])
def test_certify_outputs_fault_variants(ctx, variant):
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_batch.npz")
    B = int(g["B"])
    grp = _group(ctx, g, B)
    batch = RequestBatch.from_encoded(split_reqs(g))
    r = grp.certify_outputs(batch, g[f"{variant}_outputs"])
    assert np.array_equal(r["selected"], g[f"{variant}_sel"].astype(np.uint32))
    assert np.array_equal(r["satisfied"], g[f"{variant}_sat"].astype(bool))
    assert np.array_equal(r["label"], g[f"{variant}_label"])
    assert np.array_equal(r["r_roots"], g[f"{variant}_r_roots"])
    assert int(r["manifest_len"][0]) == int(g[f"{variant}_mlen"])
    assert np.array_equal(r["a_root"], g[f"{variant}_a_root"])


def test_certify_batch_invariant(ctx):
    """Batch == sequential (tests/test_engine.cpp:134-150): certifying a
    request alone gives the same leaf hashes as inside the batch."""
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_batch.npz")
    B = int(g["B"])
    grp = _group(ctx, g, B)
    reqs = split_reqs(g)
    full = grp.certify(RequestBatch.from_encoded(reqs), want_leaves=True)
    for k in (0, 5, B - 1):
        one = grp.certify(RequestBatch.from_encoded([reqs[k]]), want_leaves=True)
        assert np.array_equal(one["leaf_hashes"][:, 0], full["leaf_hashes"][:, k])


def test_ingest_ahead_and_out_of_order(ctx):
    """Tickets ingested ahead certify to the same results in any order; a
    full ring is an error, not a hang."""
    from paper_2205_15757_b200 import InvalidArgument, RequestBatch
    g = golden("c1_batch.npz")
    grp = _group(ctx, g, int(g["B"]))
    reqs = split_reqs(g)
    b = RequestBatch.from_encoded(reqs)
    half = RequestBatch.from_encoded(reqs[:6])
    want = grp.certify(b)
    want_half = grp.certify(half)
    ring = 24  # cg_group ingest ring depth (CG_INGEST_RING)
    t = [grp.ingest(b if i % 2 == 0 else half) for i in range(ring)]
    with pytest.raises(InvalidArgument):
        grp.ingest(b)
    order = [(5 * i + 3) % ring for i in range(ring)]  # a permutation
    for i in order:
        r = grp.certify_ticket(t[i])
        w = want if i % 2 == 0 else want_half
        assert np.array_equal(r["a_root"], w["a_root"]) and np.array_equal(r["r_roots"], w["r_roots"])
    assert np.array_equal(want["a_root"], g["honest_a_root"])


def test_fetch_ticket_after_next_certify(ctx):
    """Batch i's results stay readable (fetch_ticket) while batch i+1 is
    certified: per-batch results live in the batch's ingest slot."""
    from paper_2205_15757_b200 import RequestBatch
    g = golden("c1_batch.npz")
    grp = _group(ctx, g, int(g["B"]))
    b = RequestBatch.from_encoded(split_reqs(g))
    t0, t1 = grp.ingest(b), grp.ingest(b)
    grp.certify_ticket(t0, sync=False)
    grp.certify_ticket(t1, sync=False)
    r0 = grp.fetch_ticket(t0)
    r1 = grp.fetch_ticket(t1)
    assert np.array_equal(r0["a_root"], g["honest_a_root"])
    assert np.array_equal(r1["a_root"], g["honest_a_root"])


@pytest.mark.gpu
def test_perturbing_executor_bit_exact(ctx, oracle):
    """PerturbingExecutor on the GPU (midstate chain jobs + lane-tail kernel)
    vs the compiled reference's outputs (golden) and the oracle: bit-exact
    for the fp64 linear model; for softmax models (exp within 4 ulp of glibc)
    the offsets applied to the GPU's own unperturbed outputs are bit-exact."""
    from paper_2205_15757_b200 import CudaExecutor, InvalidArgument, Model, PerturbingExecutor
    g = golden("perturb.npz")
    for c in range(int(g["ncases"])):
        u, v, sm, node = (int(t) for t in g[f"c{c}_case"])
        mag = float(g[f"c{c}_mag"])
        dig = g[f"c{c}_digest"].tobytes()
        m = Model.load_linear(ctx, g[f"c{c}_file"].tobytes(), dig)
        x = g[f"c{c}_inputs"]
        y = PerturbingExecutor(ctx, node, mag).run(m, x)
        if not sm:
            assert np.array_equal(y, g[f"c{c}_outputs"]), c
        plain = CudaExecutor(ctx).run(m, x)
        want = np.stack([oracle.perturb(node, dig, x[k], plain[k], mag) for k in range(len(x))])
        assert np.array_equal(y, want), c
        m.free()
    # larger batch, every tail shape (u mod 8 sweeps P mod 64), random nodes
    from oracle.oracle import Reference  # noqa: F401  (oracle only checks)
    rng = np.random.default_rng(9)
    for u in (2, 3, 8, 9, 15, 16, 100, 777):
        v = int(rng.integers(1, 40))
        W = rng.normal(size=(v, u)) / np.sqrt(u)
        b = rng.normal(size=v) * 0.1
        import hashlib, struct
        f = struct.pack(">QQ?", u, v, False) + struct.pack(">I", v * u) + \
            W.astype(">f8").tobytes() + struct.pack(">I", v) + b.astype(">f8").tobytes()
        dig = hashlib.sha256(f).digest()
        m = Model.load_linear(ctx, f, dig)
        x = rng.uniform(-1, 1, (33, u))
        node = int(rng.integers(0, 2**63))
        y = PerturbingExecutor(ctx, node, 0.01).run(m, x)
        plain = CudaExecutor(ctx).run(m, x)
        want = np.stack([oracle.perturb(node, dig, x[k], plain[k], 0.01) for k in range(33)])
        assert np.array_equal(y, want), u
        with pytest.raises(InvalidArgument):
            ctx._check(ctx.L.cg_exec_run_perturbed(ctx.h, m.h, None, 0, 0, None, 0, 0,
                                                   __import__("ctypes").c_double(-1.0)))
        m.free()


@pytest.mark.gpu
@pytest.mark.parametrize("mag", [1e-9, 0.02])
def test_certify_batch_perturbed(ctx, oracle, mag):
    """The reference harness wraps node i's executor in
    PerturbingExecutor(node_index=i, perturb_magnitude) (harness.cpp:255-258,
    default 1e-9). Certified outputs == the compiled reference's outputs
    (golden) plus the oracle's offsets for provider p, bit-exact; agreement,
    leaves and roots == certifying those outputs as precomputed replica
    outputs (that path is itself pinned to the reference's certify_batch)."""
    from paper_2205_15757_b200 import InvalidArgument, RequestBatch
    g = golden("c1_batch.npz")
    B, N = int(g["B"]), int(g["N"])
    grp = _group(ctx, g, B)
    with pytest.raises(InvalidArgument):
        grp.set_perturbation(-1.0)
    grp.set_perturbation(mag)
    batch = RequestBatch.from_encoded(split_reqs(g))
    r = grp.certify(batch, want_outputs=True, want_leaves=True)
    want = np.stack([np.stack([oracle.perturb(p, g["digests"][p].tobytes(), g["inputs"][k],
                                              g["outputs"][p, k], mag) for k in range(B)])
                     for p in range(N)])
    assert not np.array_equal(want, g["outputs"])
    assert np.array_equal(r["outputs"], want)
    ref = _group(ctx, g, B).certify_outputs(batch, want, want_leaves=True)
    for key in ("selected", "diameter", "satisfied", "label", "r_roots", "a_root",
                "manifest_len", "leaf_hashes"):
        assert np.array_equal(r[key], ref[key]), key
    grp.set_perturbation(0.0)
    r0 = grp.certify(batch, want_outputs=True)
    assert np.array_equal(r0["outputs"], g["outputs"])


@pytest.mark.gpu
def test_encode_results_payload(ctx, oracle):
    """encode_results (messages.cpp:48-50): the device-encoded PREPARE
    result payload == u32be count || the oracle's InferenceResult encodings
    (pinned by the golden R-leaf hashes) of the golden outputs, per provider."""
    from oracle.oracle import parse_request
    from paper_2205_15757_b200 import InvalidArgument, RequestBatch
    g = golden("c1_batch.npz")
    B, N = int(g["B"]), int(g["N"])
    grp = _group(ctx, g, B)
    with pytest.raises(InvalidArgument):
        grp.encode_results(0)  # nothing certified yet
    reqs = split_reqs(g)
    grp.certify(RequestBatch.from_encoded(reqs))
    gid = g["gid"].tobytes()
    for p in range(N):
        want = B.to_bytes(4, "big") + b"".join(
            oracle.result_encode(parse_request(reqs[k])["request_id"], p, gid, 1,
                                 g["outputs"][p, k], g["digests"][p].tobytes())
            for k in range(B))
        assert grp.encode_results(p) == want
    with pytest.raises(InvalidArgument):
        grp.encode_results(N)
