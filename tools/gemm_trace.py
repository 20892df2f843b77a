"""Per-tile timeline of CTA 0 for 1x1 conv GEMM shapes (dev tool).
python tools/gemm_trace.py  -> time, achieved TB/s and per-tile event deltas."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
f = ctx.L.cg_dbg_gemm_trace
names = ["prod_start", "prod_got_stage", "mma_got_tmem", "mma_got_data", "mma_commit",
         "epi_got_acc", "epi_w2_done", "epi_w9_done"]
shapes = [("stage1 c3 K64 N256 +res", 401408, 256, 64, 1),
          ("stage1 ds K64 N256", 401408, 256, 64, 0),
          ("stage1 c1 K256 N64", 401408, 64, 256, 0),
          ("stage3 c3 K256 N1024 +res", 25088, 1024, 256, 1)]
for name, M, N, K, res in shapes:
    for BN in (64, 128, 256):
        if BN > N:
            continue
        tr = np.zeros(16 * 64, np.int64)
        us = C.c_double()
        rc = f(ctx.h, M, N, K, BN, res, tr.ctypes.data_as(C.c_void_p), C.byref(us))
        assert rc == 0
        byts = M * K * 2 + M * N * 2 * (2 if res else 1)
        t = tr.reshape(16, 64)
        n = int((t[0] > 0).sum())
        t = t[:, :n] - t[0, 0]
        per_tile = np.diff(t[6]).mean() if n > 2 else 0
        print(f"{name:28s} BN={BN:3d}: {us.value:7.1f} us  {byts / us.value / 1e6:5.2f} TB/s  "
              f"tiles/CTA {n}  cycles/tile {per_tile:7.0f}")
        if BN == 128 or N == 64:
            for i in range(min(n, 5)):
                print("   tile", i, {nm: int(t[j, i]) for j, nm in enumerate(names)})
