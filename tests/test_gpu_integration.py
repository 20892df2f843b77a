"""GPU: drop-in proof. The reference's own InferenceEngine (unmodified,
compiled from /root/reference into oracle/_ref) executes batches through
CudaExecutor (include/credo_gpu_adapters.hpp) and must produce results
bit-identical to its stock ToyExecutor; gpu_select_quorum and batched
hashing must equal distance::select_quorum and merkle::leaf_hash."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
DEMO = os.path.join(ROOT, "oracle", "_ref", "integration_demo")


def test_reference_engine_with_cuda_executor():
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built (needs /root/reference at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 mismatches" in out.stdout


CNN_DEMO = os.path.join(ROOT, "oracle", "_ref", "integration_cnn")


def test_reference_requests_certified_on_every_gpu(tmp_path):
    """The headline path as a drop-in: a C++ program linking the UNMODIFIED
    reference builds a ModelGroup of 3 ResNet-50 descriptors (params["arch"],
    files fetched by the reference's filesystem_fetcher), signs requests with
    make_signed_request, checks them with verify_request, and certifies them
    through GroupServer (load_group -> batch former -> dispatch) on every
    visible GPU from ONE process; the certificates must be identical across
    GPUs and equal to the reference's own recomputation from the GPU outputs."""
    import torch
    if not os.path.exists(CNN_DEMO):
        pytest.skip("oracle/_ref/integration_cnn not built (needs /root/reference at build time)")
    from paper_2205_15757_b200.workload import resnet_group
    files, digs, _ = resnet_group("resnet50", replicas=3, seed=0, jitter=5e-3)
    for p, f in enumerate(files):
        (tmp_path / f"m{p}.bin").write_bytes(f)
        (tmp_path / f"m{p}.arch").write_text("resnet50\n")
    ndev = min(2, torch.cuda.device_count())
    out = subprocess.run([CNN_DEMO, str(tmp_path), "3", "8"] + [str(d) for d in range(ndev)],
                         capture_output=True, text=True, timeout=900)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert f"{ndev} device(s)" in out.stdout and " 0 mismatches" in out.stdout


SCENARIO = os.path.join(ROOT, "oracle", "_ref", "integration_scenario")


def test_run_scenario_with_gpu_executor():
    """§8(f)3 live integration: the reference's own simulated cluster
    (run_scenario, N=4, f=1, PBFT ordering, proxies, clients) with every
    node's ToyExecutor running on the GPU (CudaExecutor, wired at link time
    where harness.cpp:255 builds executors): no deadlock, every request
    certified, check_invariants() empty, and the rendered trace byte-identical
    to the stock CPU run -- for the honest, agree_then_execute, corrupt-beyond
    and corrupt-within-epsilon scenarios of tests/test_harness.cpp and a
    C1-shaped (3072 -> 10) workload. Then the reference's strategy benchmark
    (bench_strategies, experiments.cpp:60-80) with the GPU executor under the
    default, the measured LinearToyModel and the measured ResNet-50 batch
    cost: every request certified under both strategies."""
    if not os.path.exists(SCENARIO):
        pytest.skip("oracle/_ref/integration_scenario not built (needs /root/reference at build time)")
    # device time of one ResNet-50 replica's forward at batch 1 and 4 (the
    # harness's exec_batch_max) -> the ExecCost the strategy benchmark uses
    import ctypes as C
    from paper_2205_15757_b200 import Context, Model
    from paper_2205_15757_b200.workload import resnet_group
    ctx = Context(0)
    files, digs, _ = resnet_group("resnet50", replicas=1, seed=0)
    m = Model.load_cnn(ctx, files[0], digs[0])
    ms = {}
    for b in (1, 4):
        v = C.c_double()
        assert ctx.L.cg_dbg_forward_bench(ctx.h, m.h, b, 20, C.byref(v)) == 0
        ms[b] = v.value
    per_item = max(0.0, (ms[4] - ms[1]) / 3.0) * 1e3
    fixed = max(1.0, ms[1] * 1e3 - per_item)
    m.free()
    ctx.close()
    out = subprocess.run([SCENARIO, str(round(fixed)), str(round(per_item))], capture_output=True,
                         text=True, timeout=1200)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout
    assert out.stdout.count("all certified 1") == 6


VERIFY = os.path.join(ROOT, "oracle", "_ref", "integration_verify")


def test_certificate_assembly_and_verification_batched():
    """§8(f)1: certificate assembly and verification at batch scale
    (include/credo_gpu_certs.hpp over cg_cert_leaf_hashes). On every node's
    ordered slots of run_scenario (honest, agree_then_execute, corrupt
    beyond / within epsilon, C1 and ImageNet shapes), assemble_responses
    must equal the reference's assemble_response (proxy.cpp:80-186) for
    every op, and verify_responses must equal verify_response
    (certificate.cpp:325-347) on every certified response and on forged
    variants of each (flipped output, path sibling/side, attestation kind,
    signatures, duplicate attestor, dropped result, failure reason, primary
    root, altered request) -- genuine ones accepted, every forgery rejected."""
    if not os.path.exists(VERIFY):
        pytest.skip("oracle/_ref/integration_verify not built (needs /root/reference at build time)")
    out = subprocess.run([VERIFY], capture_output=True, text=True, timeout=1200)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout
