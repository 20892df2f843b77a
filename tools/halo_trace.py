"""CTA-0 timeline of a halo-mode 3x3 conv (cg_dbg_halo_trace): per tile the
producer start, MMA start (accumulator free), first halo ready, MMA
committed, epilogue start and end (clock64 cycles relative to the first
event). Dev tool.

  python tools/halo_trace.py [B H C N BN]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

B, H, Cc, N, BN = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (128, 56, 64, 64, 64)))
PAIR = int(sys.argv[6]) if len(sys.argv) > 6 else 0
ctx = Context(0)
tr = np.zeros(16 * 64, np.int64)
us = C.c_double()
rc = ctx.L.cg_dbg_halo_trace2(ctx.h, B, H, Cc, N, BN, PAIR, tr.ctypes.data_as(C.c_void_p),
                              C.byref(us))
assert rc == 0, rc
tr = tr.reshape(16, 64)
t0 = tr[tr > 0].min()
flops = 2.0 * B * H * H * 9 * Cc * N
print(f"B={B} H={H} C={Cc} N={N} BN={BN} pair={PAIR}: {us.value:.1f} us, "
      f"{flops / us.value / 1e6:.0f} TFLOP/s")
names = ["prod", "p_load", "mma_go", "data", "mma_done", "epi_go", "epi_end2", "epi_end9"]
print("tile " + " ".join(f"{n:>9s}" for n in names) + "  | end of epilogue warps 2..9 - t0")
for i in range(12):
    print(f"{i:4d} " + " ".join(f"{(tr[s, i] - t0) if tr[s, i] else -1:9d}" for s in range(8))
          + " | " + " ".join(f"{(tr[8 + w, i] - t0) if tr[8 + w, i] else -1:6d}" for w in range(8)))
