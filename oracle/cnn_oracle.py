"""TEST INFRASTRUCTURE — CPU forward oracle for the CNN replica executor.

The reference has no CNN execution path (its SPEC.md:8 replaces ONNX/ImageNet
models with LinearToyModel, proj/src/model.cpp:12-36), so forward parity at
ImageNet shapes is UNPINNED by reference tests: this restatement is
torchvision's fp32 eval-mode forward of the same state dict (BN unfolded).
Only tests/, smoke() and bench.py's cpu legs may use it.
"""
from __future__ import annotations

import numpy as np


def build(arch: str, state_dict):
    import torchvision
    m = getattr(torchvision.models, arch)(weights=None).eval()
    m.load_state_dict(state_dict)
    return m


def logits(model, inputs: np.ndarray, image: int = 224) -> np.ndarray:
    """inputs: (B, 3*image*image) f64 CHW rows -> (B, classes) f32 logits."""
    import torch
    x = torch.from_numpy(np.ascontiguousarray(inputs, np.float64)).float()
    x = x.view(-1, 3, image, image)
    with torch.no_grad():
        return model(x).numpy()


def softmax_f64(lg: np.ndarray) -> np.ndarray:
    """LinearToyModel's softmax (model.cpp:26-34) applied to f32 logits
    widened to f64, summed in index order."""
    y = lg.astype(np.float64)
    y = np.exp(y - y.max(-1, keepdims=True))
    out = np.empty_like(y)
    for i in range(y.shape[0]):
        s = 0.0
        for v in y[i]:
            s += v
        out[i] = y[i] / s
    return out
