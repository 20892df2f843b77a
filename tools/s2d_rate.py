"""Timing + CTA-0 per-tile timeline of the s2d stem GEMM (conv1 7x7/2 as 16
taps of K = 16) at the C2 shape (3 grouped replicas x 128 images, 224 px).
Dev tool: python tools/s2d_rate.py [B] [reps]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
names = ["prod", "ld0_w2", "mma_go", "data", "commit", "epi_go", "epi_end2", "epi_end9"]
tr = np.zeros(16 * 64, np.int64)
us = C.c_double()
rc = ctx.L.cg_dbg_s2d_trace(ctx.h, B, 224, reps, tr.ctypes.data_as(C.c_void_p), C.byref(us))
assert rc == 0, rc
Gs = 115
rows = reps * B * Gs * Gs
tiles = reps * ((B * Gs * Gs + 255) // 256)
fl = 2.0 * reps * B * 112 * 112 * 64 * 147
byt = rows * 32 + rows * 128
print(f"s2d stem B={B} reps={reps}: {us.value:.1f} us, {fl / us.value / 1e6:.0f} TF/s (7x7 FLOPs), "
      f"{byt / us.value / 1e6:.2f} TB/s (A + grid out), {tiles} tiles, "
      f"MMA floor (48 cyc x 32 / tile, 148 SMs, 1.9 GHz) {tiles * 32 * 48 / 148 / 1.9e3:.1f} us")
t = tr.reshape(16, 64)
n = int((t[0] > 0).sum())
c = t[4, :n]
print(f"tiles traced {n}, commit-to-commit {np.diff(c).mean() if n > 2 else 0:.0f} cyc, "
      f"epi_go-to-epi_go {np.diff(t[5, :n]).mean() if n > 2 else 0:.0f} cyc")
t0 = t[t > 0].min()
print("tile " + " ".join(f"{x:>8s}" for x in names) + "  | end of epilogue warps 2..9 - epi_go")
for i in range(min(n, 12)):
    print(f"{i:4d} " + " ".join(f"{(t[j, i] - t0) if t[j, i] else -1:8d}" for j in range(8)) + " | "
          + " ".join(f"{t[8 + w, i] - t[5, i]:6d}" for w in range(8)))
