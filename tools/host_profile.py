"""Host-side cost of the pipelined certify loop (dev tool)."""
import os
import sys
import time
from collections import deque

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import U, make_group  # noqa: E402
from paper_2205_15757_b200 import Context  # noqa: E402
from paper_2205_15757_b200.workload import signed_requests  # noqa: E402

ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
B = 128
grp, models, *_ = make_group(ctx, B)
b = signed_requests(B, U, seed=1)
d = torch.from_numpy(b.inputs).cuda()
from copy import copy  # noqa: E402
db = copy(b)
db.inputs, db.B, db.u = d.data_ptr(), B, U
D = 6
pend = deque(grp.ingest(db) for _ in range(D))
for _ in range(5):
    grp.certify_ticket(pend.popleft(), sync=False)
    pend.append(grp.ingest(db))
torch.cuda.synchronize()
ti = tc = 0.0
K = 20
t0 = time.perf_counter()
for _ in range(K):
    a = time.perf_counter()
    grp.certify_ticket(pend.popleft(), sync=False)
    c = time.perf_counter()
    pend.append(grp.ingest(db))
    e = time.perf_counter()
    tc += c - a
    ti += e - c
host = time.perf_counter() - t0
torch.cuda.synchronize()
gpu = time.perf_counter() - t0
print(f"per step: certify enqueue {1e3 * tc / K:.2f} ms, ingest {1e3 * ti / K:.2f} ms, "
      f"host total {1e3 * host / K:.2f} ms, wall incl. drain {1e3 * gpu / K:.2f} ms")
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    grp.certify_ticket(pend.popleft(), sync=False)
    pend.append(grp.ingest(db))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
