"""Grouped vs per-replica forward inside certify (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import EUCLIDEAN, Context, CudaExecutor, Model, ModelGroup  # noqa
from paper_2205_15757_b200.workload import resnet_group, signed_requests  # noqa

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = Context(0)
files, digs, _ = resnet_group("resnet50", replicas=3)
models = [Model.load_cnn(ctx, f, d) for f, d in zip(files, digs)]
grp = ModelGroup(ctx, models, 1, EUCLIDEAN, 0.1, b"group-0", 1, max_batch=B)
batch = signed_requests(B, 3 * 224 * 224, seed=9)
r = grp.certify(batch, want_outputs=True)
ex = CudaExecutor(ctx)
for p in range(3):
    y = ex.run(models[p], batch.inputs)
    d = np.abs(r["outputs"][p] - y)
    print(p, "max abs diff", d.max(), "argmax equal", np.array_equal(y.argmax(-1), r["outputs"][p].argmax(-1)),
          "max |log ratio|", np.abs(np.log(np.maximum(y, 1e-300)) - np.log(np.maximum(r["outputs"][p], 1e-300))).max())
