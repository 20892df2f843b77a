"""Synthetic workloads in the reference's own recipes (no datasets, no
checkpoints exist offline).

* :func:`resnet_group` — a model group of jittered random-init ResNets,
  following harness::generate_group (reference proj/src/harness.cpp:346-395):
  one shared base (torchvision init under ``torch.manual_seed(seed)``, BN in
  eval mode with its default running stats) plus independent per-replica
  uniform jitter, sized so honest replicas agree well inside epsilon.
* :func:`cnn_model_file` — the canonical CNN model file whose
  SHA-256 is the descriptor's weights_digest (include/credo/domain.hpp:62-73).
* :func:`signed_requests` — the run_scenario client (harness.cpp:449-458,
  564-575): inputs U(-1,1), nonce = u64 counter || u64 rng, request_id =
  H(client_pub || 0x1F || nonce) (domain.cpp:238-241), Ed25519 signature over
  H(0x01 || body) (domain.cpp:177-202).
"""
from __future__ import annotations

import ctypes as C
import glob
import hashlib
import struct

import numpy as np

from .credo import RequestBatch

CNN_MAGIC = b"credo.cnn.v1"


def _str(b: bytes) -> bytes:
    return struct.pack(">I", len(b)) + b


def cnn_model_file(arch: str, state_dict, input_dim: int, output_dim: int,
                   softmax: bool = True) -> bytes:
    """str magic | str arch | u64 in | u64 out | bool softmax | u32 n |
    n × {str name | u32 ndim | u64 dims | u32 count | f32 BE...} (sorted)."""
    parts = [_str(CNN_MAGIC), _str(arch.encode()),
             struct.pack(">QQB", input_dim, output_dim, int(softmax))]
    names = sorted(k for k in state_dict if not k.endswith("num_batches_tracked"))
    parts.append(struct.pack(">I", len(names)))
    for k in names:
        t = state_dict[k].detach().float().contiguous().cpu().numpy()
        parts.append(_str(k.encode()))
        parts.append(struct.pack(">I", t.ndim) + b"".join(struct.pack(">Q", d) for d in t.shape))
        parts.append(struct.pack(">I", t.size))
        parts.append(t.astype(">f4").tobytes())
    return b"".join(parts)


def resnet_state_dicts(arch: str = "resnet50", replicas: int = 3, seed: int = 0,
                       jitter: float = 5e-3, salt: int = 0):
    """Shared base + per-replica jitter U(±jitter · mean|w|) on every conv/fc
    weight (the generate_group recipe; BN statistics stay shared)."""
    import torch
    import torchvision
    torch.manual_seed(seed)
    base = getattr(torchvision.models, arch)(weights=None).eval().state_dict()
    out = []
    for r in range(replicas):
        g = torch.Generator().manual_seed(1_000_003 * (salt + 1) + r)
        sd = {}
        for k, v in base.items():
            if v.dtype.is_floating_point and k.endswith("weight") and v.dim() in (2, 4):
                sd[k] = v + (torch.rand(v.shape, generator=g) * 2 - 1) * jitter * v.abs().mean()
            else:
                sd[k] = v.clone()
        out.append(sd)
    return out


def resnet_group(arch: str = "resnet50", replicas: int = 3, seed: int = 0,
                 jitter: float = 5e-3, image: int = 224, classes: int = 1000,
                 softmax: bool = True, salt: int = 0):
    """Returns (files, digests, state_dicts)."""
    sds = resnet_state_dicts(arch, replicas, seed, jitter, salt)
    files = [cnn_model_file(arch, sd, 3 * image * image, classes, softmax) for sd in sds]
    return files, [hashlib.sha256(f).digest() for f in files], sds


CNN_ARCHS = ("resnet50", "resnet101", "resnet152", "vgg16", "mobilenet_v2")
HETERO_GROUP = ("resnet50", "resnet101", "vgg16", "mobilenet_v2")  # BASELINE configs[2]


def hetero_group(archs=HETERO_GROUP, seed: int = 0, image: int = 224, classes: int = 1000,
                 softmax: bool = True):
    """A heterogeneous model group: replica p is architecture archs[p]
    (torchvision init under torch.manual_seed(seed + p), eval BN).
    Returns (files, digests, state_dicts)."""
    import torch
    import torchvision
    files, sds = [], []
    for p, arch in enumerate(archs):
        if arch not in CNN_ARCHS:
            raise ValueError(f"unsupported architecture {arch}")
        torch.manual_seed(seed + p)
        sd = getattr(torchvision.models, arch)(weights=None).eval().state_dict()
        sds.append(sd)
        files.append(cnn_model_file(arch, sd, 3 * image * image, classes, softmax))
    return files, [hashlib.sha256(f).digest() for f in files], sds


def _sodium():
    for p in glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/pyzmq.libs/libsodium*.so*"):
        try:
            L = C.CDLL(p)
            if L.sodium_init() >= 0:
                return L
        except OSError:
            pass
    return None


def signed_requests(B: int, u: int, seed: int = 1, group_id: bytes = b"group-0",
                    eps=None, inputs: np.ndarray | None = None):
    """B requests as a RequestBatch (+ their canonical encodings' framing)."""
    rng = np.random.default_rng(seed)
    if inputs is None:
        inputs = rng.uniform(-1.0, 1.0, (B, u))
    L = _sodium()
    pk = C.create_string_buffer(32)
    sk = C.create_string_buffer(64)
    seed_bytes = hashlib.sha256(b"client-key" + struct.pack(">Q", seed)).digest()
    if L is not None:
        L.crypto_sign_seed_keypair(pk, sk, seed_bytes)
        pub = pk.raw
    else:
        pub = hashlib.sha256(seed_bytes).digest()
    ids, pubs, nonces, sigs = [], [], [], []
    for i in range(B):
        nonce = struct.pack(">QQ", i, int(rng.integers(0, 2**63)))
        rid = hashlib.sha256(pub + b"\x1f" + nonce).digest()
        e = None if eps is None else eps[i]
        body = (rid + _str(group_id) + struct.pack(">I", u) +
                inputs[i].astype(">f8").tobytes() +
                (b"\x00" if e is None else b"\x01" + struct.pack(">d", e)) +
                pub + _str(nonce))
        dig = hashlib.sha256(b"\x01" + body).digest()
        if L is not None:
            sig = C.create_string_buffer(64)
            L.crypto_sign_detached(sig, None, dig, C.c_ulonglong(32), sk)
            sig = sig.raw
        else:
            sig = hashlib.sha512(sk.raw + dig).digest()
        ids.append(np.frombuffer(rid, np.uint8))
        pubs.append(np.frombuffer(pub, np.uint8))
        nonces.append(nonce)
        sigs.append(np.frombuffer(sig, np.uint8))
    return RequestBatch(np.stack(ids), np.ascontiguousarray(inputs, np.float64),
                        np.stack(pubs), nonces, np.stack(sigs), eps)


def encode_request(batch: RequestBatch, k: int, group_id: bytes = b"group-0") -> bytes:
    """InferenceRequest::encode bytes of request k (domain.cpp:144-158)."""
    x = np.asarray(batch.inputs[k], np.float64)
    e = None if batch.eps is None else batch.eps[k]
    return (batch.request_ids[k].tobytes() + _str(group_id) +
            struct.pack(">I", x.size) + x.astype(">f8").tobytes() +
            (b"\x00" if e is None else b"\x01" + struct.pack(">d", e)) +
            batch.client_pubs[k].tobytes() + _str(batch.nonces[k]) +
            batch.client_sigs[k].tobytes())
