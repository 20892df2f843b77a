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
