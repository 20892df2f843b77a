"""Probe: certify one batch through an N-replica LinearToyModel group on one
GPU (C4's N=8, f=2 shape at C1 model size) to separate the N=8 certify path
from the CNN forwards. Usage: python tools/n8_probe.py N B"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup  # noqa: E402
from paper_2205_15757_b200.workload import signed_requests  # noqa: E402

N, B = int(sys.argv[1]), int(sys.argv[2])
u, v = 3072, 10
rng = np.random.default_rng(0)
import hashlib, struct  # noqa: E402,E401
ctx = Context(0)
ms = []
W0 = rng.normal(size=(v, u)) / np.sqrt(u)
for p in range(N):
    W = W0 + rng.uniform(-1e-6, 1e-6, W0.shape)
    b = np.zeros(v)
    f = struct.pack(">QQ?", u, v, False) + struct.pack(">I", v * u) + W.astype(">f8").tobytes() + \
        struct.pack(">I", v) + b.astype(">f8").tobytes()
    ms.append(Model.load_linear(ctx, f, hashlib.sha256(f).digest()))
g = ModelGroup(ctx, ms, (N - 1) // 3, EUCLIDEAN, 0.1, b"group-0", 1, max_batch=B, topk=5)
batch = signed_requests(B, u, seed=3)
t = time.time()
r = g.certify(batch)
print("N", N, "B", B, "certify s", round(time.time() - t, 3), "satisfied",
      int(np.sum(r["satisfied"])), flush=True)
