"""Probe of the C4 configuration on one GPU with timestamps per phase:
model-file generation, loads, one synchronous certify, then a pipelined loop,
for one version and then both live versions. Memory after each phase.

    python tools/c4_probe.py [replicas] [batch] [steps]
"""
import faulthandler
import sys
import time

faulthandler.dump_traceback_later(600, exit=True)

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup  # noqa: E402
from paper_2205_15757_b200.workload import resnet_group, signed_requests  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
K = int(sys.argv[3]) if len(sys.argv) > 3 else 6
T0 = time.time()


def log(*a):
    free, tot = torch.cuda.mem_get_info()
    print(f"[{time.time() - T0:7.1f}s] used {(tot - free) / 2**30:6.1f} GiB |", *a, flush=True)


torch.cuda.set_device(0)
ctx = Context(0)
groups = []
for version, salt in ((1, 0), (2, 1000)):
    files, digs, _ = resnet_group("resnet50", replicas=N, seed=0, jitter=5e-3, salt=salt)
    log(f"v{version}: {N} model files generated")
    ms = []
    for f, d in zip(files, digs):
        t = time.time()
        ms.append(Model.load_cnn(ctx, f, d))
        log(f"  loaded replica {len(ms) - 1} in {time.time() - t:.2f}s")
    del files
    g = ModelGroup(ctx, ms, (N - 1) // 3, EUCLIDEAN, 0.1, b"group-0", version, max_batch=B, topk=5)
    groups.append((g, ms))
    log(f"v{version}: group created")

batch = signed_requests(B, 3 * 224 * 224, seed=7)
d = torch.from_numpy(batch.inputs).to("cuda:0")
import copy  # noqa: E402
db = copy.copy(batch)
db.inputs, db.B, db.u = d.data_ptr(), B, 3 * 224 * 224
for vi, (g, _) in enumerate(groups):
    t = time.time()
    r = g.certify(db)
    log(f"v{vi + 1}: sync certify {time.time() - t:.2f}s satisfied {int(np.sum(r['satisfied']))}/{B}")
for live in ([0], [0, 1]):
    from collections import deque
    pend = {v: deque() for v in live}
    D = 4
    for j in range(D):
        for v in live:
            pend[v].append(groups[v][0].ingest(db))
    torch.cuda.synchronize()
    t = time.time()
    for i in range(K):
        ts = time.time()
        for v in live:
            groups[v][0].certify_ticket(pend[v].popleft(), sync=False)
            pend[v].append(groups[v][0].ingest(db))
        torch.cuda.synchronize()
        log(f"live {live}: step {i} {time.time() - ts:.3f}s")
    for v in live:
        while pend[v]:
            groups[v][0].certify_ticket(pend[v].popleft(), sync=False)
    ctx.join()
    torch.cuda.synchronize()
    dt = time.time() - t
    log(f"live {live}: {K} steps {dt:.2f}s -> {K * B / dt:.0f} req/s (synchronised steps)")
for g, ms in groups:
    g.free()
    for m in ms:
        m.free()
log("done")
