"""Cycles per back-to-back SS-mode tcgen05 MMA (K=16) for N = 64 / 128 /
256: M=128 on one SM (one or two accumulators, 1 or 148 CTAs), and M=256 on
an SM pair (cta_group::2, 2 or 148 CTAs). The tcgen05 floor is
max(M,128)*N/(256*cta_group) cycles per dispatch (B300_MICROARCH.md)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
for N in (64, 128, 256):
    for ctas, mode, label in ((148, 0, "M=128 1 SM  "), (148, 1, "M=128 2 accs"),
                              (2, 2, "M=256 pair  "), (148, 2, "M=256 pairs ")):
        c = C.c_double()
        rc = ctx.L.cg_dbg_mma_rate(ctx.h, N, 4096, ctas, mode, C.byref(c))
        assert rc == 0, rc
        work = 2 if mode == 2 else 1
        print(f"N={N:3d} {label} ctas={ctas:3d}: {c.value:6.1f} cycles/MMA "
              f"({c.value / work:5.1f} per 128-row slab)")
