"""GPU: the heterogeneous model group of BASELINE configs[2] (ResNet-50,
ResNet-101, VGG-16, MobileNetV2, one replica each): every new architecture's
forward against the torchvision fp32 CPU oracle (same stated tolerance as
tests/test_gpu_cnn.py), batch invariance, and whole-group certification with
every decision and digest recomputed by the oracle from the GPU outputs."""
import numpy as np
import pytest
from conftest import check_certificate

pytestmark = pytest.mark.gpu

B_TEST = 4
U = 3 * 224 * 224


@pytest.fixture(scope="module")
def hetero(ctx):
    from paper_2205_15757_b200 import Model
    from paper_2205_15757_b200.workload import HETERO_GROUP, hetero_group
    files, digs, sds = hetero_group(HETERO_GROUP, seed=11)
    models = [Model.load_cnn(ctx, f, d) for f, d in zip(files, digs)]
    yield dict(archs=HETERO_GROUP, files=files, digests=digs, sds=sds, models=models)
    for m in models:
        m.free()


@pytest.mark.parametrize("p", [0, 1, 2, 3])
def test_forward_logits_vs_cpu_oracle(ctx, hetero, p):
    """Raw logits (model file with softmax off) against torchvision fp32.
    Stated tolerance (bf16 weights/activations, fp32 accumulation):
    max|Δlogit| <= 0.03 * max|logit| and correlation >= 0.999 over the batch,
    top-1 equal wherever the CPU top-2 margin exceeds 5% of max|logit|."""
    from oracle import cnn_oracle
    from paper_2205_15757_b200 import CudaExecutor, Model
    from paper_2205_15757_b200.workload import cnn_model_file
    import hashlib
    arch = hetero["archs"][p]
    f = cnn_model_file(arch, hetero["sds"][p], U, 1000, softmax=False)
    m = Model.load_cnn(ctx, f, hashlib.sha256(f).digest())
    rng = np.random.default_rng(20 + p)
    x = rng.uniform(-1, 1, (B_TEST, U))
    lg_gpu = CudaExecutor(ctx).run(m, x)
    m.free()
    lg = cnn_oracle.logits(cnn_oracle.build(arch, hetero["sds"][p]), x).astype(np.float64)
    scale = np.abs(lg).max()
    err = np.abs(lg_gpu - lg).max() / scale
    corr = np.corrcoef(lg_gpu.ravel(), lg.ravel())[0, 1]
    print(f"{arch}: max|dlogit|/max|logit| {err:.4f}, corr {corr:.6f}, max|logit| {scale:.3g}")
    assert err <= 0.03 and corr >= 0.999
    top2 = np.sort(lg, -1)[:, -2:]
    sure = (top2[:, 1] - top2[:, 0]) > 0.05 * scale
    assert np.array_equal(np.argmax(lg_gpu, -1)[sure], np.argmax(lg, -1)[sure])


@pytest.mark.parametrize("p", [2, 3])
def test_batch_invariant(ctx, hetero, p):
    from paper_2205_15757_b200 import CudaExecutor
    rng = np.random.default_rng(30 + p)
    x = rng.uniform(-1, 1, (3, U))
    ex = CudaExecutor(ctx)
    full = ex.run(hetero["models"][p], x)
    one = ex.run(hetero["models"][p], x[2:3])
    assert np.array_equal(one[0], full[2])


def test_hetero_group_certify(ctx, hetero, oracle):
    """4 replicas, f = 1, each replica a different architecture; the
    per-replica loop runs every model on its own input operand."""
    from paper_2205_15757_b200 import EUCLIDEAN, CudaExecutor, ModelGroup
    from paper_2205_15757_b200.workload import signed_requests
    gid = b"group-h"
    grp = ModelGroup(ctx, hetero["models"], 1, EUCLIDEAN, 0.05, gid, 1, max_batch=8, topk=5)
    batch = signed_requests(B_TEST, U, seed=6, group_id=gid, eps=[None, 1e-4, None, 0.5])
    r = grp.certify(batch, want_outputs=True, want_leaves=True)
    sels, sats = check_certificate(r, batch, hetero["digests"], 1, 0.05, gid, oracle)
    assert not sats[1]  # a tiny epsilon cannot be met by four different nets
    ex = CudaExecutor(ctx)
    for p, m in enumerate(hetero["models"]):  # certify's forwards == exec_run's
        assert np.array_equal(r["outputs"][p], ex.run(m, batch.inputs))
    grp.free()
