"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol
include/credo_gpu.h declares. No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HDR = os.path.join(ROOT, "include", "credo_gpu.h")
LIB = os.path.join(ROOT, "paper_2205_15757_b200", "libcredo_gpu.so")


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|uint64_t|void\*)\s+\**(cg_\w+)\(",
                                 txt, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("cg_sha256_batch", "cg_select_quorum_batch", "cg_exec_run",
              "cg_certify_batch", "cg_merkle_root_batch", "cg_model_load_cnn",
              "cg_exec_run_perturbed"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("libcredo_gpu.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    if not os.path.exists(LIB):
        pytest.fail("libcredo_gpu.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_gpu_context_fails_loudly():
    """Without a B200 the product refuses to run (no CPU fallback)."""
    import paper_2205_15757_b200 as p
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(p.CredoError):
        p.Context(0)


def test_library_loaded_before_torch():
    """libcredo_gpu.so resolves libnccl.so.2 to the copy torch uses, so
    loading it first must not break a later `import torch` (the two NCCL
    builds export different symbol sets)."""
    import subprocess
    import sys
    from paper_2205_15757_b200.credo import LIB_PATH
    code = f"import ctypes; ctypes.CDLL({LIB_PATH!r}); import torch; print('ok')"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
