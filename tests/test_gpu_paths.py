"""GPU: Merkle authentication paths for certificate assembly / verification
(Tree::auth_path and get_merkle_root, merkle.cpp:69-93,
as used by assemble_response proxy.cpp:80-186 and verify_cert
certificate.cpp:215-288) against the compiled reference."""
import numpy as np
import pytest
from conftest import golden, split_reqs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 100, 1000])
def test_auth_paths_match_reference(ctx, oracle, n):
    from oracle.oracle import Reference
    R = Reference()
    rng = np.random.default_rng(n)
    leaves = [rng.integers(0, 256, int(rng.integers(1, 90)), dtype=np.uint8).tobytes()
              for _ in range(n)]
    lh = [oracle.leaf_hash(x) for x in leaves]
    idx = list(range(n)) if n <= 13 else sorted(rng.choice(n, 40, replace=False).tolist())
    paths, root = ctx.auth_paths(lh, idx)
    assert root == oracle.merkle_root(lh)
    for i, p in zip(idx, paths):
        assert p == R.auth_path(leaves, i), i
        assert R.path_root(leaves[i], p) == root
    got = ctx.path_roots([lh[i] for i in idx], paths)
    assert all(r == root for r in got)
    if n > 1:  # a forged sibling no longer reaches the root
        bad = [list(p) for p in paths]
        s, d = bad[0][0]
        bad[0][0] = (bytes([s[0] ^ 1]) + s[1:], d)
        assert ctx.path_roots([lh[idx[0]]], bad[:1])[0] != root


def test_auth_path_bad_index(ctx, oracle):
    from paper_2205_15757_b200 import InvalidArgument
    lh = [oracle.leaf_hash(b"x%d" % i) for i in range(4)]
    with pytest.raises(InvalidArgument):
        ctx.auth_paths(lh, [4])
    with pytest.raises(InvalidArgument):
        ctx.auth_paths([], [])


def test_group_paths_rebuild_certificate_roots(ctx, oracle):
    """verify_cert's two proofs from the GPU's paths: the ordering proof
    (result leaf -> provider's R root) and the trust proof (whole-batch or
    single attestation leaf -> attestor's A root)."""
    from oracle.oracle import Reference
    from paper_2205_15757_b200 import EUCLIDEAN, Model, ModelGroup, RequestBatch
    R = Reference()
    g = golden("c1_batch.npz")
    N, B, gid = int(g["N"]), int(g["B"]), g["gid"].tobytes()
    models = [Model.load_linear(ctx, g["files"][p].tobytes(), g["digests"][p].tobytes())
              for p in range(N)]
    grp = ModelGroup(ctx, models, 1, EUCLIDEAN, float(g["eps"]), gid, 1, max_batch=B, topk=3)
    encs = split_reqs(g)
    batch = RequestBatch.from_encoded(encs)
    from copy import deepcopy

    from paper_2205_15757_b200.workload import encode_request
    tight = deepcopy(batch)
    tight.eps = list(tight.eps)
    tight.eps[2] = 1e-12  # an unsatisfiable epsilon: a failure leaf for request 2
    kinds = set()
    for variant, b in (("honest", batch), ("partial_fault", batch), ("failure", tight)):
        outs = g[f"{variant}_outputs"]
        r = grp.certify_outputs(b, outs)
        encs = [encode_request(b, k, gid) for k in range(B)]
        for p in range(N):
            paths = grp.auth_paths(p, range(B))
            for k in range(B):
                res = oracle.result_encode(batch.request_ids[k].tobytes(), p, gid, 1,
                                           outs[p, k], g["digests"][p].tobytes())
                leaf = b"\x52" + encs[k] + res
                assert R.path_root(leaf, paths[k]) == r["r_roots"][p].tobytes(), (p, k)
        m = int(r["manifest_len"][0])
        apaths = grp.auth_paths(N, range(m))
        roots = ctx.path_roots([r["a_leaf_hashes"][i].tobytes() for i in range(m)], apaths)
        assert all(x == r["a_root"].tobytes() for x in roots)
        kinds |= set(int(x) for x in r["manifest_kind"])
    assert kinds == {0, 1, 2}, kinds  # whole-batch, single and failure leaves
    grp.free()
