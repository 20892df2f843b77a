"""Generates the committed golden fixtures from the COMPILED REFERENCE
(oracle/_ref/libcredo_ref.so, built from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py

Outputs tests/golden/*.npz. Nothing at test time reads /root/reference; the
fixtures carry the reference's own answers so the GPU box can check against
them. Fixture contents:

* sha256.npz     — KATs ("", "abc", FIPS 448-bit, 1e6 x 'a') + random lengths
* merkle.npz     — Tree::build roots over 1..40 random leaves
* quorum.npz     — select_quorum + ensemble_label on random instances
                   (the test_distance.cpp:162-190 generator shape) and the
                   pinned examples of test_distance.cpp:138-154
* c1_batch.npz   — generate_group models, make_signed_request requests (some
                   with epsilon overrides), LinearToyModel outputs, leaf
                   hashes, and ref_certify_batch results for three fault
                   patterns (honest / one replica corrupt on some requests /
                   tight epsilon -> failures)
* c1_full.npz    — the same at SURVEY §8(d)'s C1 shape (3072 -> 10 softmax,
                   3 models, batch 64, seed 7), every-5th-request fault
* c1_misfit.npz  — a batch with two wrong-input-dimension requests
                   (missing_result_leaf, unsatisfied, failure leaves)
* c1_slot.npz    — a mixed op list: ok / rejected requests, activate_group
                   ops (0x52 / 0x4D / 0x47 R leaves, explicit failure leaves)
* perturb.npz    — PerturbingExecutor(ToyExecutor, node, magnitude) outputs
                   over generate_group models with u in {1, 9, 3072} (0, 1
                   and 384 shared SHA blocks; 1- and 2-block lane tails), a
                   softmax model, several nodes and magnitudes

    python tests/golden/make_golden.py perturb   # that fixture alone
    python tests/golden/make_golden.py c1_full   # that fixture alone
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference, parse_linear_model_file  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha_fixture(R):
    rng = np.random.default_rng(0x5A)
    msgs = [b"", b"abc",
            b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq"]
    lens = list(range(0, 140)) + [183, 184, 191, 192, 255, 256, 1000, 4099]
    for n in lens:
        msgs.append(rng.integers(0, 256, n, dtype=np.uint8).tobytes())
    digests = [R.sha256(m) for m in msgs]
    million_a = R.sha256(b"a" * 1000000)
    lens_arr = np.array([len(m) for m in msgs], np.uint64)
    np.savez_compressed(os.path.join(OUT, "sha256.npz"),
                        data=np.frombuffer(b"".join(msgs) or b"\0", np.uint8),
                        lens=lens_arr,
                        digests=np.frombuffer(b"".join(digests), np.uint8).reshape(-1, 32),
                        million_a=np.frombuffer(million_a, np.uint8))


def merkle_fixture(R):
    rng = np.random.default_rng(0x3E)
    all_leaves, counts, roots, leaf_hashes = [], [], [], []
    for n in list(range(1, 41)) + [64, 65, 127]:
        leaves = [rng.integers(0, 256, int(rng.integers(1, 80)), dtype=np.uint8).tobytes()
                  for _ in range(n)]
        roots.append(R.merkle_root(leaves))
        leaf_hashes.extend(R.leaf_hash(x) for x in leaves)
        all_leaves.extend(leaves)
        counts.append(n)
    np.savez_compressed(
        os.path.join(OUT, "merkle.npz"),
        leaf_data=np.frombuffer(b"".join(all_leaves), np.uint8),
        leaf_lens=np.array([len(x) for x in all_leaves], np.uint64),
        leaf_hashes=np.frombuffer(b"".join(leaf_hashes), np.uint8).reshape(-1, 32),
        counts=np.array(counts, np.uint64),
        roots=np.frombuffer(b"".join(roots), np.uint8).reshape(-1, 32))


def quorum_fixture(R):
    """Random instances in the shape of test_distance.cpp:162-190 (n=4..8,
    f=(n-1)/3, present >= n-f, dim 1 or 4, 30% wide spread) plus v=10/1000
    softmax-like vectors, all three metrics, and the pinned examples."""
    rng = np.random.default_rng(0xD157)
    rows = []
    V = 16
    for trial in range(2000):
        n = int(rng.integers(3, 9))
        f = max(1, (n - 1) // 3) if n > 3 else 1
        present_n = (n - f) + int(rng.integers(0, f + 1))
        dim = int(rng.choice([1, 4, 10, 16]))
        metric = int(rng.choice([0, 0, 2] + ([1] if dim == 1 else [])))
        ids = rng.permutation(n)[:present_n]
        center = rng.uniform(-1, 1, dim)
        outs = np.zeros((8, V))
        mask = 0
        for i in ids:
            spread = 5.0 if rng.random() < 0.3 else 0.05
            outs[i, :dim] = center + rng.uniform(-spread, spread, dim)
            mask |= 1 << int(i)
        eps = float(rng.uniform(0, 0.3))
        idx = np.array(sorted(int(i) for i in ids), np.uint64)
        sm, sd, ss = R.select_quorum(outs[idx][:, :dim], idx, n, f, metric, eps)
        lab = R.ensemble_label(outs[:n, :dim], sm, f) if ss else -1
        rows.append((n, f, dim, metric, mask, eps, outs, sm, sd, ss, lab))
    # pinned examples (test_distance.cpp:138-154), scalars, n=4 f=1
    for vals, eps in (([1.00, 1.01, 1.02, 5.0], 0.2), ([2.0] * 4, 0.0),
                      ([1.0, 1.5, 2.0, 2.5], 0.2)):
        outs = np.zeros((8, V))
        outs[:4, 0] = vals
        idx = np.arange(4, dtype=np.uint64)
        sm, sd, ss = R.select_quorum(outs[:4, :1], idx, 4, 1, 0, eps)
        lab = R.ensemble_label(outs[:4, :1], sm, 1) if ss else -1
        rows.append((4, 1, 1, 0, 0xF, eps, outs, sm, sd, ss, lab))
    cols = list(zip(*rows))
    np.savez_compressed(
        os.path.join(OUT, "quorum.npz"),
        n=np.array(cols[0], np.uint32), f=np.array(cols[1], np.uint32),
        dim=np.array(cols[2], np.uint32), metric=np.array(cols[3], np.uint32),
        present=np.array(cols[4], np.uint32), eps=np.array(cols[5]),
        outs=np.stack(cols[6]), selected=np.array(cols[7], np.uint64),
        diameter=np.array(cols[8]), satisfied=np.array(cols[9], np.uint8),
        label=np.array(cols[10], np.int64))


def c1_fixture(R):
    u, v, N, B, eps = 512, 10, 3, 12, 0.05
    gid = b"group-0"
    files, digs = R.generate_group(gid, u, v, N, 0, eps, seed=7, softmax=False)
    inputs, encs = R.make_requests(1, 7, B, u, gid)
    # re-sign a few requests with epsilon overrides (opt(eps) present)
    rng = np.random.default_rng(11)
    for k in (3, 7):
        encs[k] = R.make_request(1, bytes(rng.integers(0, 256, 16, dtype=np.uint8)),
                                 gid, inputs[k], eps=0.5)
    outs = np.stack([R.linear_run(files[p], inputs, v) for p in range(N)])  # N,B,v
    leaf = np.zeros((N, B, 32), np.uint8)
    for p in range(N):
        for k in range(B):
            leaf[p, k] = np.frombuffer(
                R.result_leaf_hash(encs[k], p, gid, 1, outs[p, k], digs[p]), np.uint8)
    variants = {}
    # honest
    variants["honest"] = outs.copy()
    # replica 2 corrupt (+1.0 on every lane, corrupt_result) on requests 1,4,9
    bad = outs.copy()
    for k in (1, 4, 9):
        bad[2, k] += 1.0
    variants["partial_fault"] = bad
    # replicas 1 and 2 both corrupt on request 5 -> unsatisfied -> failure leaf
    fail = bad.copy()
    fail[1, 5] -= 2.0
    variants["failure"] = fail
    res = {}
    h = R.batch_new(encs, 1)
    for name, o in variants.items():
        r = R.certify_batch(h, N, 1, 0, eps, o, 1, digs, threads=1)
        r2 = R.certify_batch(h, N, 1, 0, eps, o, 1, digs, threads=4)
        assert r["a_root"] == r2["a_root"] and r["r_roots"] == r2["r_roots"]
        res[name] = r
    R.batch_free(h)
    save = dict(u=u, v=v, N=N, B=B, eps=eps, gid=np.frombuffer(gid, np.uint8),
                files=np.stack([np.frombuffer(f_, np.uint8) for f_ in files]),
                digests=np.stack([np.frombuffer(d, np.uint8) for d in digs]),
                req_lens=np.array([len(e) for e in encs], np.uint64),
                reqs=np.frombuffer(b"".join(encs), np.uint8),
                inputs=inputs, outputs=outs, leaf_hashes=leaf)
    for name, o in variants.items():
        r = res[name]
        save[f"{name}_outputs"] = o
        save[f"{name}_sel"] = r["sel_mask"]
        save[f"{name}_diam"] = r["diameter"]
        save[f"{name}_sat"] = r["satisfied"]
        save[f"{name}_label"] = r["label"]
        save[f"{name}_r_roots"] = np.frombuffer(b"".join(r["r_roots"]), np.uint8).reshape(N, 32)
        save[f"{name}_a_root"] = np.frombuffer(r["a_root"], np.uint8)
        save[f"{name}_mlen"] = np.array(r["manifest_len"], np.uint64)
    np.savez_compressed(os.path.join(OUT, "c1_batch.npz"), **save)


def c1_full_fixture(R):
    """C1 at SURVEY §8(d)'s shape: generate_group("group-0", u=3072, v=10,
    3 models, euclidean, eps=0.05, seed=7) with softmax, requests from
    make_requests(1, 7, 64, 3072) (harness.cpp:346-395, :449-458), batch 64.
    The inputs travel inside the request encodings."""
    u, v, N, B, eps = 3072, 10, 3, 64, 0.05
    gid = b"group-0"
    files, digs = R.generate_group(gid, u, v, N, 0, eps, seed=7, softmax=True)
    inputs, encs = R.make_requests(1, 7, B, u, gid)
    outs = np.stack([R.linear_run(files[p], inputs, v) for p in range(N)])  # N,B,v
    leaf = np.zeros((N, B, 32), np.uint8)
    for p in range(N):
        for k in range(B):
            leaf[p, k] = np.frombuffer(
                R.result_leaf_hash(encs[k], p, gid, 1, outs[p, k], digs[p]), np.uint8)
    variants = {"honest": outs.copy()}
    bad = outs.copy()  # corrupt_result (+1.0 every lane) on replica 2, every 5th request
    bad[2, ::5] += 1.0
    variants["partial_fault"] = bad
    fail = bad.copy()  # replica 1 also off on request 10 -> unsatisfied -> failure leaf
    fail[1, 10] -= 2.0
    variants["failure"] = fail
    h = R.batch_new(encs, 1)
    save = dict(u=u, v=v, N=N, B=B, eps=eps, gid=np.frombuffer(gid, np.uint8),
                files=np.stack([np.frombuffer(f_, np.uint8) for f_ in files]),
                digests=np.stack([np.frombuffer(d, np.uint8) for d in digs]),
                req_lens=np.array([len(e) for e in encs], np.uint64),
                reqs=np.frombuffer(b"".join(encs), np.uint8), outputs=outs, leaf_hashes=leaf)
    for name, o in variants.items():
        r = R.certify_batch(h, N, 1, 0, eps, o, 1, digs, threads=4)
        save[f"{name}_outputs"] = o
        save[f"{name}_sel"] = r["sel_mask"]
        save[f"{name}_diam"] = r["diameter"]
        save[f"{name}_sat"] = r["satisfied"]
        save[f"{name}_label"] = r["label"]
        save[f"{name}_r_roots"] = np.frombuffer(b"".join(r["r_roots"]), np.uint8).reshape(N, 32)
        save[f"{name}_a_root"] = np.frombuffer(r["a_root"], np.uint8)
        save[f"{name}_mlen"] = np.array(r["manifest_len"], np.uint64)
    R.batch_free(h)
    np.savez_compressed(os.path.join(OUT, "c1_full.npz"), **save)


def c1_misfit_fixture(R):
    """A C1-model batch (u=512) with two misfit requests (input dims 500 and
    513): execute_batch skips them (engine.cpp:286-291), so every R tree has
    missing_result_leaf there and try_attest leaves them unsatisfied."""
    u, v, N, B, eps = 512, 10, 3, 12, 0.05
    gid = b"group-0"
    files, digs = R.generate_group(gid, u, v, N, 0, eps, seed=7, softmax=False)
    inputs, encs = R.make_requests(1, 9, B, u, gid)
    rng = np.random.default_rng(13)
    misfit = {4: 500, 9: 513}
    dims = np.full(B, u, np.uint64)
    rows = [inputs[k] for k in range(B)]
    for k, d in misfit.items():
        rows[k] = rng.uniform(-1, 1, d)
        dims[k] = d
        encs[k] = R.make_request(1, bytes(rng.integers(0, 256, 16, dtype=np.uint8)), gid, rows[k])
    outs = np.zeros((N, B, v))
    fit = [k for k in range(B) if k not in misfit]
    for p in range(N):
        outs[p, fit] = R.linear_run(files[p], np.stack([rows[k] for k in fit]), v)
    miss = np.array([k in misfit for k in range(B)], np.uint8)
    h = R.batch_new(encs, 1)
    r = R.certify_batch(h, N, 1, 0, eps, outs, 1, digs, threads=1, missing=miss)
    r4 = R.certify_batch(h, N, 1, 0, eps, outs, 1, digs, threads=4, missing=miss)
    assert r["a_root"] == r4["a_root"] and r["r_roots"] == r4["r_roots"]
    R.batch_free(h)
    save = dict(u=u, v=v, N=N, B=B, eps=eps, gid=np.frombuffer(gid, np.uint8), dims=dims,
                missing=miss, files=np.stack([np.frombuffer(f_, np.uint8) for f_ in files]),
                digests=np.stack([np.frombuffer(d, np.uint8) for d in digs]),
                req_lens=np.array([len(e) for e in encs], np.uint64),
                reqs=np.frombuffer(b"".join(encs), np.uint8), outputs=outs,
                sel=r["sel_mask"], diam=r["diameter"], sat=r["satisfied"], label=r["label"],
                r_roots=np.frombuffer(b"".join(r["r_roots"]), np.uint8).reshape(N, 32),
                a_root=np.frombuffer(r["a_root"], np.uint8),
                mlen=np.array(r["manifest_len"], np.uint64))
    np.savez_compressed(os.path.join(OUT, "c1_misfit.npz"), **save)


SLOT_KINDS = [0, 0, 1, 0, 2, 0, 0, 2, 0, 1, 0, 0]
SLOT_REASONS = ["", "", "unknown group version", "", "", "", "", "group op rejected: retired",
                "", "malformed request", "", ""]


def c1_slot_fixture(R):
    """A mixed PRE-PREPARE op list on the C1 models (u=512): ok requests,
    two requests the primary rejected (no result: missing_result_leaf; A leaf
    = their failure record with the reason) and two activate_group ops (R leaf
    group_op_leaf; one rejected, with a failure leaf) -- build_result_tree
    (messages.cpp:235-258) and the try_attest manifest with outcomes only for
    the ok request ops. Also an empty slot's roots (noop leaf)."""
    u, v, N, eps = 512, 10, 3, 0.05
    gid = b"group-0"
    files, digs = R.generate_group(gid, u, v, N, 0, eps, seed=7, softmax=False)
    B = len(SLOT_KINDS)
    inputs, encs_all = R.make_requests(1, 11, B, u, gid)
    encs = [encs_all[k] if SLOT_KINDS[k] <= 1 else b"" for k in range(B)]
    outs = np.zeros((N, B, v))
    req = [k for k in range(B) if SLOT_KINDS[k] <= 1]
    for p in range(N):
        outs[p, req] = R.linear_run(files[p], inputs[req], v)
    outs[2, 5] += 1.0  # one faulty provider on one op: no whole-batch leaf for 2
    r = R.certify_slot(encs, SLOT_KINDS, SLOT_REASONS, N, 1, eps, outs, 1, digs)
    save = dict(u=u, v=v, N=N, B=B, eps=eps, gid=np.frombuffer(gid, np.uint8),
                kinds=np.array(SLOT_KINDS, np.uint8), inputs=inputs,
                files=np.stack([np.frombuffer(f_, np.uint8) for f_ in files]),
                digests=np.stack([np.frombuffer(d, np.uint8) for d in digs]),
                req_lens=np.array([len(e) for e in encs], np.uint64),
                reqs=np.frombuffer(b"".join(encs), np.uint8), outputs=outs,
                entry_lens=np.array([len(e) for e in r["entries"]], np.uint64),
                entries=np.frombuffer(b"".join(r["entries"]), np.uint8),
                rec_lens=np.array([len(e) for e in r["records"]], np.uint64),
                recs=np.frombuffer(b"".join(r["records"]) or b"\0", np.uint8),
                sat=r["satisfied"],
                r_roots=np.frombuffer(b"".join(r["r_roots"]), np.uint8).reshape(N, 32),
                a_root=np.frombuffer(r["a_root"], np.uint8),
                mlen=np.array(r["manifest_len"], np.uint64))
    np.savez_compressed(os.path.join(OUT, "c1_slot.npz"), **save)


# (u, v, softmax, node, magnitude, seed)
PERTURB_CASES = [(1, 3, False, 0, 0.25, 11), (9, 5, False, 3, 1e-3, 12),
                 (3072, 10, False, 1, 0.05, 7), (3072, 10, True, 2, 1e-4, 7),
                 (40, 17, False, 2**40 + 5, 3.5, 13), (3072, 10, False, 0, 0.0, 7)]


def perturb_fixture(R):
    save = {}
    for c, (u, v, sm, node, mag, seed) in enumerate(PERTURB_CASES):
        files, digs = R.generate_group(b"group-0", u, v, 1, 0, 0.05, seed, softmax=sm)
        x = np.random.default_rng(100 + c).uniform(-1, 1, (6, u))
        save[f"c{c}_file"] = np.frombuffer(files[0], np.uint8)
        save[f"c{c}_digest"] = np.frombuffer(digs[0], np.uint8)
        save[f"c{c}_inputs"] = x
        save[f"c{c}_plain"] = R.linear_run(files[0], x, v)
        save[f"c{c}_outputs"] = R.perturbing_run(files[0], x, v, node, mag)
        save[f"c{c}_case"] = np.array([u, v, int(sm), node], np.uint64)
        save[f"c{c}_mag"] = np.array(mag, np.float64)
    save["ncases"] = np.array(len(PERTURB_CASES))
    np.savez_compressed(os.path.join(OUT, "perturb.npz"), **save)


if __name__ == "__main__":
    if not Reference.available():
        sys.exit("oracle/_ref/libcredo_ref.so missing: run `make -C oracle ref` "
                 "where /root/reference exists")
    R = Reference()
    if sys.argv[1:] == ["perturb"]:
        perturb_fixture(R)
        sys.exit(0)
    if sys.argv[1:] == ["c1_full"]:
        c1_full_fixture(R)
        sys.exit(0)
    if sys.argv[1:] == ["c1_misfit"]:
        c1_misfit_fixture(R)
        sys.exit(0)
    if sys.argv[1:] == ["c1_slot"]:
        c1_slot_fixture(R)
        sys.exit(0)
    sha_fixture(R)
    merkle_fixture(R)
    quorum_fixture(R)
    c1_fixture(R)
    c1_full_fixture(R)
    c1_misfit_fixture(R)
    c1_slot_fixture(R)
    perturb_fixture(R)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
