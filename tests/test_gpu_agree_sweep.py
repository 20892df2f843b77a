"""C5 agreement sweep on the GPU: the throughput form of select_quorum +
ensemble_label + compact label digests (cg_agree_device, one thread per
request) bit-exact against the oracle on device-generated synthetic
outputs, both metrics, n in {4, 8}, v in {10, 1000}; and the host API's
large-batch route equals its small-batch (CTA-per-request) route."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _sweep(ctx, seed, R, n, f, v, metric, eps_choices, shift=0.1):
    dev = torch.device("cuda:0")
    outs = torch.empty(n * R * v, dtype=torch.float64, device=dev)
    ids = torch.empty(R * 32, dtype=torch.uint8, device=dev)
    ctx.synth_outputs(seed, R, n, v, 0.05, shift, outs.data_ptr(), ids.data_ptr())
    rng = np.random.default_rng(seed)
    eps = torch.from_numpy(rng.choice(eps_choices, R)).to(dev)
    sel = torch.empty(R, dtype=torch.int32, device=dev)
    diam = torch.empty(R, dtype=torch.float64, device=dev)
    sat = torch.empty(R, dtype=torch.uint8, device=dev)
    st = torch.empty(R, dtype=torch.int8, device=dev)
    lab = torch.empty(R, dtype=torch.int64, device=dev)
    dig = torch.empty(R * 32, dtype=torch.uint8, device=dev)
    ctx.agree_device(outs.data_ptr(), R * v, v, eps.data_ptr(), R, n, f, v, metric,
                     sel.data_ptr(), diam.data_ptr(), sat.data_ptr(), st.data_ptr(),
                     lab.data_ptr(), ids.data_ptr(), 5, dig.data_ptr())
    ctx.synchronize()
    got = dict(selected=sel.cpu().numpy().view(np.uint32), diameter=diam.cpu().numpy(),
               satisfied=sat.cpu().numpy().astype(bool), label=lab.cpu().numpy(),
               digest=dig.cpu().numpy().reshape(R, 32), status=st.cpu().numpy())
    host = (outs.cpu().numpy().reshape(n, R, v), ids.cpu().numpy().reshape(R, 32),
            eps.cpu().numpy())
    return got, host


@pytest.mark.parametrize("n,f,v,metric", [(8, 2, 1000, 0), (4, 1, 1000, 0), (8, 2, 10, 0),
                                          (4, 1, 10, 2), (8, 3, 1000, 2), (3, 1, 10, 0),
                                          (4, 1, 7, 0)])
def test_agree_device_bit_exact(ctx, oracle, n, f, v, metric):
    R = 6000  # above the throughput-form threshold (kAgreeRowsMinBatch = 4096)
    # generator eps 0.05: honest euclidean spread ~0.005, faulty ~0.15;
    # chebyshev: honest <= 0.05/(4 sqrt v), faulty ~0.15/sqrt v
    s = np.sqrt(v)
    eps_choices = [0.05, 0.003, 0.5] if metric == 0 else [0.005 / s, 0.05 / s, 0.3 / s]
    got, (outs, ids, eps) = _sweep(ctx, 100 + n + v, R, n, f, v, metric, eps_choices)
    want = oracle.agree_batch(outs, f, metric, eps, ids, version=5)
    assert not got["status"].any()
    for key in ("selected", "diameter", "satisfied", "label", "digest"):
        assert np.array_equal(got[key], want[key]), key
    # the sweep exercises every decision kind
    assert got["satisfied"].any() and (~got["satisfied"]).any()
    assert (got["selected"][got["satisfied"]] != (1 << n) - 1).any()


def test_agree_small_batch_route_matches(ctx, oracle):
    """Below the threshold cg_agree_device uses the CTA-per-request kernel
    plus the standalone digest kernel: same answers."""
    got, (outs, ids, eps) = _sweep(ctx, 7, 700, 8, 2, 100, 0, [0.05, 0.003, 0.5])
    want = oracle.agree_batch(outs, 2, 0, eps, ids, version=5)
    for key in ("selected", "diameter", "satisfied", "label", "digest"):
        assert np.array_equal(got[key], want[key]), key


def test_host_select_quorum_large_batch(ctx, oracle):
    rng = np.random.default_rng(3)
    R, n, v = 5000, 4, 16
    outs = rng.random((R, n, v))
    outs[rng.random((R, n)) < 0.15] += 0.3
    eps = rng.choice([0.9, 1.2], R)
    big = ctx.select_quorum_batch(outs, n, 1, 0, eps)
    small = [ctx.select_quorum_batch(outs[i:i + 1000], n, 1, 0, eps[i:i + 1000])
             for i in range(0, R, 1000)]
    for key in ("selected", "diameter", "satisfied", "label"):
        assert np.array_equal(big[key], np.concatenate([s[key] for s in small])), key
    want = oracle.agree_batch(np.transpose(outs, (1, 0, 2)), 1, 0, eps)
    assert np.array_equal(big["selected"], want["selected"])
    assert np.array_equal(big["label"], want["label"])


def test_label_digest_batch(ctx, oracle):
    rng = np.random.default_rng(4)
    ids = rng.integers(0, 256, (300, 32), dtype=np.uint8)
    labels = rng.integers(-1, 1000, 300)
    got = ctx.label_digests(ids, labels, 11)
    for k in range(300):
        assert got[k].tobytes() == oracle.label_digest(ids[k].tobytes(), 11, int(labels[k]))


def _adversarial(rng, R, n, v):
    from adversarial import adversarial
    return adversarial(rng, R, n, v)


@pytest.mark.parametrize("n,f,v,metric", [(4, 1, 6, 0), (8, 2, 6, 0), (5, 1, 4, 2),
                                          (8, 3, 3, 2), (3, 1, 1, 1)])
def test_agreement_adversarial_both_kernels(ctx, oracle, n, f, v, metric):
    """Bit-exact against the oracle on NaN/Inf/tie cases, through both the
    CTA-per-request kernel (small batch) and the thread-per-request kernel
    (large batch); the oracle's select_quorum follows distance.cpp's exact
    comparison semantics (std::max, strict '>' against epsilon)."""
    rng = np.random.default_rng(n * 100 + v)
    R = 5000
    outs = _adversarial(rng, R, n, v)
    eps = rng.choice([0.0, 0.1, 0.25, 1.0], R)
    want = oracle.agree_batch(np.transpose(outs, (1, 0, 2)), f, metric, eps)
    big = ctx.select_quorum_batch(outs, n, f, metric, eps)               # wide kernel
    small = ctx.select_quorum_batch(outs[:300], n, f, metric, eps[:300])  # CTA kernel
    for key in ("selected", "satisfied", "label"):
        assert np.array_equal(big[key], want[key]), key
        assert np.array_equal(small[key], want[key][:300]), key
    assert np.array_equal(big["diameter"].view(np.uint64), want["diameter"].view(np.uint64))
    assert np.array_equal(small["diameter"].view(np.uint64),
                          want["diameter"][:300].view(np.uint64))
