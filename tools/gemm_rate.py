"""(residual flag bit 1 = SM pair)
Mainloop throughput of the identity-row conv GEMM on compute-bound shapes
vs torch.mm (cuBLAS) bf16 on the same shapes, plus CTA-0's per-tile timeline.
Dev tool: python tools/gemm_rate.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
import torch  # noqa: E402

f = ctx.L.cg_dbg_gemm_trace_mode
names = ["prod", "p_stage", "mma_go", "data", "commit", "epi_go", "epi_end2", "epi_end9"]
shapes = [("square K2048", 32768, 2048, 2048, 256, 0),
          ("square K2048 BN128", 32768, 2048, 2048, 128, 0),
          ("square K2048 pair", 32768, 2048, 2048, 256, 2),
          ("l4 c3 +res", 18816, 2048, 512, 256, 1),
          ("l4 c3 +res pair", 18816, 2048, 512, 256, 3),
          ("l4 c3 no res pair", 18816, 2048, 512, 256, 2),
          ("l4 c3 no res", 18816, 2048, 512, 256, 0),
          ("l3 c3 +res", 75264, 1024, 256, 256, 1),
          ("l3 c3 +res pair", 75264, 1024, 256, 256, 3),
          ("l3 c1 pair", 75264, 256, 1024, 256, 2),
          ("l4 c1 pair", 18816, 512, 2048, 256, 2),
          ("l3 c3 +res BN128", 75264, 1024, 256, 128, 1),
          ("l2 c3 +res", 301056, 512, 128, 256, 1),
          ("l2 c3 +res BN128", 301056, 512, 128, 128, 1),
          ("l2 c3 +res pair", 301056, 512, 128, 256, 3),
          ("l3 c1", 75264, 256, 1024, 256, 0),
          ("l3 c1 BN128", 75264, 256, 1024, 128, 0),
          ("l4 c1", 18816, 512, 2048, 256, 0),
          ("l1 c1 K64", 1204224, 64, 64, 64, 0),
          ("l1 c1 K256", 1204224, 64, 256, 64, 0),
          ("l1 c3 +res", 1204224, 256, 64, 256, 1)]
only = sys.argv[1] if len(sys.argv) > 1 else None  # run one shape (for ncu)
for label, M, N, K, BN, res in shapes:
    if only and label != only:
        continue
    tr = np.zeros(16 * 64, np.int64)
    us = C.c_double()
    rc = f(ctx.h, M, N, K, BN, res, 0, 0, tr.ctypes.data_as(C.c_void_p), C.byref(us))
    assert rc == 0, rc
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.mm(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    tus = e0.elapsed_time(e1) * 100
    fl = 2.0 * M * N * K
    t = tr.reshape(16, 64)
    n = int((t[0] > 0).sum())
    c = t[4, :n]
    per = np.diff(c).mean() if n > 2 else 0
    print(f"{label}: ours {us.value:.1f} us {fl / us.value / 1e6:.0f} TF/s | cublas {tus:.1f} us "
          f"{fl / tus / 1e6:.0f} TF/s | tiles/CTA {n}, commit-to-commit {per:.0f} cyc "
          f"(MMA floor {K // 16 * BN // 2} cyc)")
    if "l4 c3" in label or "l3 c3" in label or label.startswith("l1"):
        t0 = t[t > 0].min()
        print("tile " + " ".join(f"{x:>8s}" for x in names) + "  | end of epilogue warps 2..9 - t0")
        for i in range(min(n, 8)):
            print(f"{i:4d} " + " ".join(f"{(t[j, i] - t0) if t[j, i] else -1:8d}" for j in range(8))
                  + " | " + " ".join(f"{(t[8 + w, i] - t0) if t[8 + w, i] else -1:6d}" for w in range(8)))
    del a, b
