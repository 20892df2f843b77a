"""CTA-0 timeline of a 1x1 conv GEMM in identity vs remapped-row epilogue
(cg_dbg_gemm_trace_mode): where the per-tile time of small-K layers goes.
Dev tool: python tools/remap_trace.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
f = ctx.L.cg_dbg_gemm_trace_mode
names = ["prod", "p_stage", "mma_go", "data", "commit", "epi_go", "epi_end2", "epi_end9"]
H = 56
for label, M, N, K, BN, mode in (("l1.0 c1 K64 N64 identity", 3 * 128 * H * H, 64, 64, 64, 0),
                                 ("l1.0 c1 K64 N64 CompactToPad", 3 * 128 * H * H, 64, 64, 64, 2),
                                 ("l1.1 c1 K256 N64 CompactToPad", 3 * 128 * H * H, 64, 256, 64, 2)):
    tr = np.zeros(16 * 64, np.int64)
    us = C.c_double()
    rc = f(ctx.h, M, N, K, BN, 0, mode, H, tr.ctypes.data_as(C.c_void_p), C.byref(us))
    assert rc == 0, rc
    t = tr.reshape(16, 64)
    n = int((t[0] > 0).sum())
    t0 = t[t > 0].min()
    byts = M * K * 2 + M * N * 2
    print(f"{label}: {us.value:.1f} us ({byts / us.value / 1e6:.2f} TB/s), tiles/CTA {n}")
    print("tile " + " ".join(f"{x:>8s}" for x in names) + "  | end of epilogue warps 2..9 - t0")
    for i in range(min(n, 8)):
        print(f"{i:4d} " + " ".join(f"{(t[j, i] - t0) if t[j, i] else -1:8d}" for j in range(8))
              + " | " + " ".join(f"{(t[8 + w, i] - t0) if t[8 + w, i] else -1:6d}" for w in range(8)))
