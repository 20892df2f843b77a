"""Latency of the request-midstate SHA chains alone (one ingest of a C2
batch = B chains of 1.2 MB each, one exclusive-SM CTA per 128 requests), with
nothing else on the GPU; then k ingests at once.

  python tools/chain_latency.py [B]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2205_15757_b200 import Context  # noqa: E402
from paper_2205_15757_b200.workload import signed_requests  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = Context(0)
grp, models, *_ = bench.make_group(ctx, B)
b = signed_requests(B, bench.U, seed=5)
d = torch.from_numpy(b.inputs).cuda()
b.inputs, b.B, b.u = d.data_ptr(), B, bench.U
for k in (1, 1, 2, 4, 6):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ts = [grp.ingest(b) for _ in range(k)]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{k} ingest(s) of {B} requests: {1e3 * dt:.2f} ms wall "
          f"({1e3 * dt / (B // 128 or 1):.2f} ms per chain CTA if serial)", flush=True)
    for t_ in ts:
        grp.certify_ticket(t_, sync=False)
    torch.cuda.synchronize()
