"""Host-side cost of the e2e loop (bench.py e2e leg) per phase: submit
(structural checks + pack into pinned staging + ingest), ready, certify
enqueue, fetch. python tools/e2e_probe.py [pack_threads] [steps]"""
import sys
import time
from collections import deque

sys.path.insert(0, ".")
import numpy as np  # noqa: E402,F401
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2205_15757_b200 import Context, InferenceEngine  # noqa: E402
from paper_2205_15757_b200.workload import signed_requests  # noqa: E402

PT = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
DEPTH = int(sys.argv[3]) if len(sys.argv) > 3 else 12
B, U = 128, 3 * 224 * 224
ctx = Context(0)
grp, ms, _, _, _ = bench.make_group(ctx, B)
base = [signed_requests(B, U, seed=i) for i in range(2)]
eng = InferenceEngine(ctx, B, 10**12, pack_threads=PT)
eng.load_group(grp)
t = time.perf_counter()
reqs = [eng.prepare(signed_requests(B, U, seed=100 + i, inputs=base[i % 2].inputs), b"group-0")
        for i in range(2 * K)]
print(f"pack threads {PT}, depth {DEPTH}: signing {2 * K} batches: {time.perf_counter() - t:.1f}s", flush=True)
for rnd, lo in (("warm", 0), ("timed", K)):
    ph = dict(submit=0.0, ready=0.0, certify=0.0, fetch=0.0)
    rq, inf = deque(), deque()
    t0 = time.perf_counter()
    for i in range(K):
        a = time.perf_counter()
        eng.submit_prepared(reqs[lo + i], now_us=i)
        b = time.perf_counter()
        rq.extend(eng.ready())
        c = time.perf_counter()
        while len(rq) > DEPTH:
            g, _, tk, Bt = rq.popleft()
            g.certify_ticket(tk, sync=False, B=Bt)
            inf.append(tk)
        d = time.perf_counter()
        while len(inf) > 8:
            grp.fetch_ticket(inf.popleft())
        e = time.perf_counter()
        ph["submit"] += b - a
        ph["ready"] += c - b
        ph["certify"] += d - c
        ph["fetch"] += e - d
    while rq:
        g, _, tk, Bt = rq.popleft()
        g.certify_ticket(tk, sync=False, B=Bt)
        inf.append(tk)
    while inf:
        grp.fetch_ticket(inf.popleft())
    ctx.join()
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(rnd, f"total {1e3 * tot / K:.2f} ms/step |",
          " ".join(f"{k} {1e3 * v / K:.2f}" for k, v in ph.items()), flush=True)
eng.free()
