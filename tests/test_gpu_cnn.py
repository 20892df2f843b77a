"""GPU: the ResNet-50 replica executor (tcgen05 convs) against the CPU forward
oracle (torchvision fp32, oracle/cnn_oracle.py), and whole-group
certification of ImageNet-shaped requests.

Parity protocol: (i) per-replica outputs vs the
fp32 CPU forward within a stated bf16 tolerance; (ii) decisions and digests
bit-exact, computed by the oracle from the GPU's own per-replica outputs.

Stated tolerance (bf16 weights/activations, fp32 accumulation, 53 layers):
centred log-probability error |Δlog p - mean Δlog p| <= 0.01 * max|logit| + 0.1
per class, and top-1 agreement whenever the CPU top-2 logit margin exceeds 1.0.
"""
import numpy as np
import pytest
from conftest import check_certificate

pytestmark = pytest.mark.gpu

B_TEST = 6


@pytest.fixture(scope="module")
def r50(ctx):
    from paper_2205_15757_b200 import Model
    from paper_2205_15757_b200.workload import resnet_group
    files, digs, sds = resnet_group("resnet50", replicas=3, seed=0, jitter=5e-3)
    models = [Model.load_cnn(ctx, f, d) for f, d in zip(files, digs)]
    yield dict(files=files, digests=digs, sds=sds, models=models)
    for m in models:
        m.free()


def test_cnn_digest_mismatch_rejected(ctx, r50):
    from paper_2205_15757_b200 import DigestMismatch, Model
    bad = bytearray(r50["digests"][0])
    bad[5] ^= 0x10
    with pytest.raises(DigestMismatch):
        Model.load_cnn(ctx, r50["files"][0], bytes(bad))


def test_resnet50_forward_vs_cpu_oracle(ctx, r50):
    from oracle import cnn_oracle
    from paper_2205_15757_b200 import CudaExecutor
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (B_TEST, 3 * 224 * 224))
    p_gpu = CudaExecutor(ctx).run(r50["models"][0], x)
    lg = cnn_oracle.logits(cnn_oracle.build("resnet50", r50["sds"][0]), x)
    p_cpu = cnn_oracle.softmax_f64(lg)
    assert np.allclose(p_gpu.sum(-1), 1.0, atol=1e-12)
    d = np.log(np.maximum(p_gpu, 1e-300)) - np.log(np.maximum(p_cpu, 1e-300))
    d -= d.mean(-1, keepdims=True)
    scale = np.abs(lg).max()
    err = np.abs(d).max()
    print(f"max centred logit error {err:.4f}, max|logit| {scale:.2f}")
    assert err <= 0.01 * scale + 0.1
    top2 = np.sort(lg, -1)[:, -2:]
    sure = (top2[:, 1] - top2[:, 0]) > 1.0
    assert np.array_equal(np.argmax(p_gpu, -1)[sure], np.argmax(lg, -1)[sure])


def test_resnet50_batch_invariant(ctx, r50):
    """Same model + same input -> bit-identical output whatever the batch
    (model.hpp:45-47, tests/test_engine.cpp:134-150)."""
    from paper_2205_15757_b200 import CudaExecutor
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (5, 3 * 224 * 224))
    ex = CudaExecutor(ctx)
    full = ex.run(r50["models"][1], x)
    for k in (0, 3):
        one = ex.run(r50["models"][1], x[k:k + 1])
        assert np.array_equal(one[0], full[k])


def test_resnet50_group_certify_digests(ctx, r50, oracle):
    from paper_2205_15757_b200 import EUCLIDEAN, ModelGroup
    from paper_2205_15757_b200.workload import signed_requests
    gid = b"group-0"
    grp = ModelGroup(ctx, r50["models"], 1, EUCLIDEAN, 0.1, gid, 1, max_batch=8, topk=5)
    batch = signed_requests(B_TEST, 3 * 224 * 224, seed=5, group_id=gid,
                            eps=[None, 0.2, None, None, 0.01, None])
    r = grp.certify(batch, want_outputs=True, want_leaves=True)
    check_certificate(r, batch, r50["digests"], 1, 0.1, gid, oracle)
    grp.free()


def test_grouped_forward_equals_per_replica(ctx, r50):
    """The grouped (one launch per layer for all replicas) forward inside
    certify produces bit-identical replica outputs to exec_run per replica."""
    from paper_2205_15757_b200 import EUCLIDEAN, CudaExecutor, ModelGroup
    from paper_2205_15757_b200.workload import signed_requests
    grp = ModelGroup(ctx, r50["models"], 1, EUCLIDEAN, 0.1, b"group-0", 1, max_batch=4)
    batch = signed_requests(4, 3 * 224 * 224, seed=9)
    r = grp.certify(batch, want_outputs=True)
    ex = CudaExecutor(ctx)
    for p in range(3):
        y = ex.run(r50["models"][p], batch.inputs)
        print(p, np.abs(r["outputs"][p] - y).max(), np.argmax(y, -1), np.argmax(r["outputs"][p], -1))
        assert np.array_equal(r["outputs"][p], y)
    grp.free()
